out=gpurun_out/r2bj; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_dropin.py tests/test_stored_transforms.py tests/test_wide_layers.py -x -q -m gpu > $out/t.txt 2>&1
for c in cfg3 cfg5-yelp-gat cfg5-amazon-gat; do
  VARIANTS="a c" bash tools/ab_variants.sh $out $c 1 >> $out/ab.txt 2>&1
done
