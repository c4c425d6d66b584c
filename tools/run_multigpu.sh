#!/bin/bash
# Multi-GPU bench lines on one box (N = 2 and 4): replicas and CGP on cfg2, CGP groups on the papers-shaped cfg4.
# Usage (GPU box with >= 4 GPUs, repo root): bash tools/run_multigpu.sh [out_dir]
out=${1:-gpurun_out/multigpu}
mkdir -p "$out"
port=29600
run() {  # name, nproc, args...
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
}
run cfg2_replicas_n2 2 --no-cpu
run cfg2_replicas_n4 4 --no-cpu
run cfg2_cgp_n2 2 --no-cpu --parallel cgp
run cfg2_cgp_n4 4 --no-cpu --parallel cgp
run cfg4_cgp2_n2 2 --config cfg4
run cfg4_cgp2x2_n4 4 --config cfg4
run cfg4_cgp4_n4 4 --config cfg4 --cgp-size 4
touch "$out/failures.txt"
