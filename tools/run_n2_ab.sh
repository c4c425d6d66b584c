#!/bin/bash
# 2-GPU A/B: CGP slice sorts beside the selection (default) vs serial (OB_CGP_SERIAL=1)
out=${1:-gpurun_out/n2ab}
mkdir -p "$out"
port=29800
run() {
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
}
nvidia-smi nvlink -gt d > "$out/nvlink_before.txt" 2>&1
run cfg4_cgp2_n2 2 --config cfg4 --no-e2e
OB_CGP_SERIAL=1 run cfg4_cgp2_n2_serial 2 --config cfg4 --no-e2e
run cfg2_cgp_n2 2 --no-cpu --no-e2e --parallel cgp
OB_CGP_SERIAL=1 run cfg2_cgp_n2_serial 2 --no-cpu --no-e2e --parallel cgp
nvidia-smi nvlink -gt d > "$out/nvlink_after.txt" 2>&1
touch "$out/failures.txt"
