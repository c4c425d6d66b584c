#!/bin/bash
# Single-GPU bench lines for the other configs (cfg1, cfg3, cfg5 shapes) and an A/B of the
# wide-row aggregation slices (OB_AGG_NV_MAX=2) on the H = 512 configs.
out=${1:-gpurun_out/cfgs}
mkdir -p "$out"
for c in cfg1 cfg3; do
  timeout 900 python bench.py --config $c > "$out/$c.json" 2> "$out/$c.err"
done
for c in cfg5-yelp-gcn cfg5-yelp-gat cfg5-amazon-gcn cfg5-amazon-gat; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > "$out/$c.json" 2> "$out/$c.err"
  OB_AGG_NV_MAX=2 timeout 900 python bench.py --config $c --no-cpu --no-e2e > "$out/${c}_nv2.json" 2> "$out/${c}_nv2.err"
done
