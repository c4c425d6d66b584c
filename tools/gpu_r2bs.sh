out=gpurun_out/r2bs; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu > $out/t.txt 2>&1
VARIANTS="a e" bash tools/ab_variants.sh $out cfg5-amazon-gat 2 >> $out/ab.txt 2>&1
VARIANTS="a e" bash tools/ab_variants.sh $out cfg5-yelp-gat 1 >> $out/ab.txt 2>&1
