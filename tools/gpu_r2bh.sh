out=gpurun_out/r2bh; mkdir -p $out
for r in 1 2; do
for v in "X=1" "OB_GEMM_NO_SLABS=1" "OB_QROWS_SERIAL=1" "OB_NO_STORED_TRANSFORMS=1" "OB_SEL_CLUSTER_EDGES=4000000"; do
  env $v timeout 900 python bench.py --config cfg5-amazon-gat --no-cpu --no-e2e > $out/ag_${v}_$r.json 2>/dev/null
  python -c "
import json
d=json.loads(open('$out/ag_${v}_$r.json').read().strip().splitlines()[-1])
print('$v', $r, d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'], d['kernels_ms_per_step'])" >> $out/ab.txt
done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches_ag.csv" \
  python bench.py --config cfg5-amazon-gat --steps 2 --warmup 3 --no-cpu --no-e2e --lanes 1 > "$out/ncu.log" 2>&1
