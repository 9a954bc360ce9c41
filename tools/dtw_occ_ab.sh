# A/B of the strip refine's shared memory (query-pair copies) and CTAs per SM on C4 (serial pass)
for cfg in "16 0" "8 0" "8 3"; do
  set -- $cfg
  MESSI_DTW_QCOPIES=$1 MESSI_DTW_REFINE_OCC=$2 timeout 300 python bench.py --mode dtw --steps 2 --warmup 1 --no-cpu --latency 0 --repeats 1 > gpurun_out/occ.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/occ.log').read().strip().splitlines()[-1]);r=d['roofline']
print('K=$1 occ=$2', round(d['value'],1), 'refine_ms', round(r['refine_ms_per_step'],2), 'frac', round(r['frac'],3))"
done
