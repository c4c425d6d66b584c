# 4-GPU probe of the CGP lanes pass: PDL and hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS)
out=${1:-gpurun_out/n4probe}
mkdir -p "$out"
port=29800
run() {
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
  python -c "
import json
d=json.loads(open('$out/$name.json').read().strip().splitlines()[-1])
print('$name', d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])" >> "$out/summary.txt" 2>&1
}
run cfg2_cgp4_default 4 --no-cpu --no-e2e --parallel cgp
OB_NO_PDL=1 run cfg2_cgp4_nopdl 4 --no-cpu --no-e2e --parallel cgp
CUDA_DEVICE_MAX_CONNECTIONS=32 run cfg2_cgp4_conn32 4 --no-cpu --no-e2e --parallel cgp
run cfg2_cgp2x2_default 4 --no-cpu --no-e2e --parallel cgp --cgp-size 2
OB_NO_PDL=1 run cfg2_cgp2x2_nopdl 4 --no-cpu --no-e2e --parallel cgp --cgp-size 2
CUDA_DEVICE_MAX_CONNECTIONS=32 run cfg2_cgp2x2_conn32 4 --no-cpu --no-e2e --parallel cgp --cgp-size 2
touch "$out/failures.txt"
