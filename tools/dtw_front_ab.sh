# A/B of the best-first front bin of the DTW filter (MESSI_DTW_FRONT) with the reverse bound
run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/fab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/fab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
for F in 0.5 0.3 0.7 0.9 1.0; do MESSI_DTW_FRONT=$F run front$F; done
