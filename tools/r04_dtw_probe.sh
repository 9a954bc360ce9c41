# Round 2 (session 4): DTW critical-path probe at HEAD (skip runs give WRONG answers; timing only)
# needs a library built with -DMESSI_TIMING_KNOBS (the skip knobs are compiled out of the default build)
# and the C4 launch list (ncu, cold / serialised per-launch times)
run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/sab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/sab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
run base
MESSI_TIMING_SKIP_REFINE=1 run skip_refine
MESSI_TIMING_SKIP_FILTER=1 run skip_filter
MESSI_TIMING_SKIP_FILTER=1 MESSI_TIMING_SKIP_REFINE=1 run skip_both
MESSI_REFINE_STREAMS=4 run refine_streams4
DARGS="--mode dtw --steps 1 --warmup 3 --no-cpu --latency 0 --repeats 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r04_launches_c4.csv \
  python bench.py $DARGS > gpurun_out/ncu_launch_dtw.log 2>&1; echo "launches c4 rc=$?"
