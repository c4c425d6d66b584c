#!/bin/bash
# 2-GPU checks and bench lines: the NCCL CGP test, cfg2 CGP and replicas, papers-shaped cfg4 CGP.
out=${1:-gpurun_out/n2}
mkdir -p "$out"
timeout 900 python -m pytest tests/test_gpu_cgp.py -q -m gpu -k multi_process > "$out/pytest_nccl.txt" 2>&1
port=29700
run() {
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
}
run cfg2_cgp_n2 2 --no-cpu --parallel cgp
run cfg4_cgp2_n2 2 --config cfg4
run cfg2_replicas_n2 2 --no-cpu
touch "$out/failures.txt"
