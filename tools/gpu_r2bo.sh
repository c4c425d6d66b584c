out=gpurun_out/r2bo; mkdir -p $out
timeout 1200 python -m pytest tests -x -q -m gpu > $out/t.txt 2>&1
VARIANTS="a b" bash tools/ab_variants.sh $out cfg2 2 >> $out/ab.txt 2>&1
VARIANTS="a b" bash tools/ab_variants.sh $out cfg3 2 >> $out/ab.txt 2>&1
VARIANTS="a b" bash tools/ab_variants.sh $out cfg1 1 >> $out/ab.txt 2>&1
REPS=1000 MODES="X=1" bash tools/race_stress.sh $out
