out=gpurun_out/r2bd; mkdir -p $out
for c in cfg2 cfg3; do
for r in 1 2; do
for v in "X=1" "OB_SEL_GRID=148" "OB_SEL_GRID=74" "OB_SEL_GRID=32"; do
  env $v timeout 900 python bench.py --config $c --no-cpu --no-e2e > $out/${c}_${v}_$r.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$out/${c}_${v}_$r.json').read().strip().splitlines()[-1])
print('$c', '$v', $r, d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'], d['kernels_ms_per_step']['select'])" >> $out/ab.txt
done; done; done
