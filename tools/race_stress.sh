out=${1:-gpurun_out/stress}; mkdir -p $out
for v in ${MODES:-"X=1"}; do
  env STRESS_LANES=0 $(echo $v | tr ',' ' ') timeout 600 python tools/race_stress.py ${REPS:-1500} 1 > $out/run.log 2>&1
  echo "== $v" >> $out/summary.txt
  grep -v "^\[bench\]" $out/run.log | sort | uniq -c | sort -rn | head -12 >> $out/summary.txt
done
