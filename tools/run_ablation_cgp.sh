#!/bin/bash
# Config-5 ablation (BASELINE configs[4]): full vs srpe vs sampled on one B200 and srpe-cgp on two,
# one request at a time (--lanes 1), on a 2-GPU box.
# Usage: bash tools/run_ablation_cgp.sh [out_dir]
out=${1:-gpurun_out/ablation_cgp}
mkdir -p "$out"
port=29900
for c in cfg5-yelp-gcn cfg5-yelp-gat cfg5-amazon-gcn cfg5-amazon-gat; do
  for s in srpe sampled full; do
    CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 20 --no-cpu --no-e2e --lanes 1 --config $c \
      --strategy $s > "$out/${c}_$s.json" 2> "$out/${c}_$s.err" || echo "FAIL ${c}_$s" >> "$out/failures.txt"
  done
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 2 --steps 20 --no-cpu --no-e2e --lanes 1 --config $c --parallel cgp \
    > "$out/${c}_srpe-cgp_n2.json" 2> "$out/${c}_srpe-cgp_n2.err" || echo "FAIL ${c}_srpe-cgp" >> "$out/failures.txt"
done
touch "$out/failures.txt"
