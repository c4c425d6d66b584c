#!/bin/bash
# Round-2 closing evidence on the final commit: GPU tests, smoke, default bench line, reference arm.
out=${1:-gpurun_out/final2}
mkdir -p "$out"
timeout 1200 python -m pytest tests -q -m gpu > "$out/pytest_gpu.txt" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$out/smoke.txt" 2>&1
timeout 900 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
timeout 900 python bench.py --impl reference > "$out/bench_reference_cfg2.json" 2> "$out/bench_reference_cfg2.err"
timeout 900 python bench.py --config cfg3 > "$out/cfg3.json" 2> "$out/cfg3.err"
for c in cfg1 cfg5-yelp-gcn cfg5-yelp-gat cfg5-amazon-gcn cfg5-amazon-gat; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > "$out/$c.json" 2> "$out/$c.err"
done
