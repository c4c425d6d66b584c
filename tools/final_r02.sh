#!/bin/bash
# Round-2 final evidence on one GPU (final build): full GPU tests, smoke, default bench line,
# the reference arm, the other configs, a launch list and one ncu --set full of the aggregation.
out=${1:-gpurun_out/final}
mkdir -p "$out"
timeout 1200 python -m pytest tests -q -m gpu > "$out/pytest_gpu.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$out/smoke.txt" 2>&1
timeout 900 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$out/bench_reference_cfg2.json" 2> "$out/bench_reference_cfg2.err"
for c in cfg1 cfg3; do
  timeout 900 python bench.py --config $c > "$out/$c.json" 2> "$out/$c.err"
done
for c in cfg5-yelp-gcn cfg5-yelp-gat cfg5-amazon-gcn cfg5-amazon-gat; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > "$out/$c.json" 2> "$out/$c.err"
done
timeout 900 python bench.py --policy random --no-cpu --no-e2e > "$out/bench_cfg2_random.json" 2> "$out/bench_cfg2_random.err"
# launch list of the default single-lane request path (serialised, cold; shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches.csv" \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --lanes 1 > "$out/ncu_launches.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_agg|k_tc_gemm|k_finalize|k_select" \
  -s 60 -c 12 -o "$out/full" python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --lanes 1 > "$out/ncu_full.log" 2>&1
