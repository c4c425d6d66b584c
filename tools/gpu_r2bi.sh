out=gpurun_out/r2bi; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu > $out/t.txt 2>&1
for c in cfg3 cfg5-yelp-gat cfg5-amazon-gat; do
  VARIANTS="a b" bash tools/ab_variants.sh $out $c 2 >> $out/ab.txt 2>&1
done
