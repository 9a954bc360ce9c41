run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 $2 > gpurun_out/wab2.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/wab2.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, 'cand', round(d['stats_mean']['candidates']), 'lbk', round(d['stats_mean']['lbk_pass']), 'seedbsf', round(d['stats_mean']['seed_d2'],3))"
}
run w2000 "--window 2000"
run w1000 "--window 1000"
run w500 "--window 500"
run w4000 "--window 4000"
