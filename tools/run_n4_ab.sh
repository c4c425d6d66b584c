#!/bin/bash
# 4-GPU A/B of the CGP lanes pass: hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS) and the
# serial slice construction (OB_CGP_SERIAL=1)
out=${1:-gpurun_out/n4ab}
mkdir -p "$out"
port=29950
run() {
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
}
run cfg4_cgp4_default 4 --config cfg4 --cgp-size 4 --no-e2e
CUDA_DEVICE_MAX_CONNECTIONS=32 run cfg4_cgp4_conn32 4 --config cfg4 --cgp-size 4 --no-e2e
OB_CGP_SERIAL=1 run cfg4_cgp4_serial 4 --config cfg4 --cgp-size 4 --no-e2e
CUDA_DEVICE_MAX_CONNECTIONS=32 run cfg2_cgp4_conn32 4 --no-cpu --no-e2e --parallel cgp
touch "$out/failures.txt"
