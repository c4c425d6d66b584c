out=gpurun_out/r2bc; mkdir -p $out
for c in cfg5-amazon-gat cfg5-amazon-gcn cfg2; do
for r in 1 2; do
for v in "X=1" "OB_SEL_CLUSTER_EDGES=4000000"; do
  env $v timeout 900 python bench.py --config $c --no-cpu --no-e2e > $out/${c}_${v}_$r.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$out/${c}_${v}_$r.json').read().strip().splitlines()[-1])
print('$c', '$v', $r, d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])" >> $out/ab.txt
done; done; done
