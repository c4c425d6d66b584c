out=${1:-gpurun_out/race}; mkdir -p $out
for v in "X=1" "OB_QROWS_SERIAL=1" "CUDA_DEVICE_MAX_CONNECTIONS=8" "OB_QROWS_SERIAL=1 CUDA_DEVICE_MAX_CONNECTIONS=8" "OB_NO_PDL=1"; do
  env $v timeout 600 python -m pytest tests/test_gpu_bench_parity.py -x -q -m gpu -k "requests_vs_oracle or lanes" > $out/t.log 2>&1
  echo "$v: $(tail -1 $out/t.log)" >> $out/summary.txt
  grep -E "^E " $out/t.log | head -3 >> $out/summary.txt
done
