out=gpurun_out/r2bp; mkdir -p $out
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -m gpu -k "repeated" >> $out/t.txt 2>&1
done
REPS=3000 MODES="X=1" bash tools/race_stress.sh $out
