# A/B of the quantised LB_Keogh filter's lanes per candidate (MESSI_LBK_G) on C4
for G in 1 2 4 8 16; do
  MESSI_LBK_G=$G timeout 300 python bench.py --mode dtw --steps 2 --warmup 1 --no-cpu --latency 0 --repeats 1 > gpurun_out/lbk_$G.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/lbk_$G.log').read().strip().splitlines()[-1]);r=d['roofline']
print('G=$G', round(d['value'],1), 'lbk_ms', round(r['lbk_filter']['ms_per_step'],2), 'refine_ms', round(r['refine_ms_per_step'],2))"
done
