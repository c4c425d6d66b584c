# critical-path probe: a 30 us spin inserted after one stage (variant library "w"); p50 moves by
# ~30 us only when that stage is on the critical path
out=${OUT:-gpurun_out/whatif}; mkdir -p $out
for where in none csr qb sel qrows; do
  OB_LIB_VARIANT=w OB_WHATIF_WHERE=$where OB_WHATIF_DELAY_US=30 python bench.py --no-cpu --no-e2e --steps 30 > $out/$where.json 2> $out/$where.err
  python -c "
import json
d=json.loads(open('$out/$where.json').read().strip().splitlines()[-1])
print('$where', d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])
" >> $out/summary.txt
done
