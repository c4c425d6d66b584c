out=gpurun_out/r2bl; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu > $out/t.txt 2>&1
VARIANTS="a d" bash tools/ab_variants.sh $out cfg3 2 >> $out/ab.txt 2>&1
VARIANTS="a d" bash tools/ab_variants.sh $out cfg5-yelp-gat 1 >> $out/ab.txt 2>&1
VARIANTS="a d" bash tools/ab_variants.sh $out cfg5-amazon-gat 1 >> $out/ab.txt 2>&1
