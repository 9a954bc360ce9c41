# timing sensitivity of the DTW pipeline to each stage (answers are wrong in the skip runs)
# needs a library built with -DMESSI_TIMING_KNOBS (the skip knobs are compiled out of the default build)
run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/sab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/sab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
run base
MESSI_TIMING_SKIP_REFINE=1 run skip_refine
MESSI_TIMING_SKIP_FILTER=1 run skip_filter
MESSI_NO_REV=1 MESSI_TIMING_SKIP_REFINE=1 run norev_skip_refine
