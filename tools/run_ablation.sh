#!/bin/bash
# Config-3 gamma sweep and config-5 strategy ablation (BASELINE configs[2], configs[4]) on one B200.
# Usage (GPU box, repo root): bash tools/run_ablation.sh [out_dir]
out=${1:-gpurun_out/ablation}
mkdir -p "$out"
run() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py --steps 20 --no-cpu "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
}
for g in 0 0.05 0.1 0.2 0.3 1.0; do run cfg3_g$g --config cfg3 --gamma $g --lanes 1; done
run cfg2_policy_is --config cfg2 --policy is --no-e2e
run cfg3_policy_is --config cfg3 --policy is --no-e2e
for c in cfg5-yelp-gcn cfg5-yelp-gat cfg5-amazon-gcn cfg5-amazon-gat; do
  for s in srpe sampled full; do run ${c}_$s --config $c --strategy $s --no-e2e --lanes 1; done
done
