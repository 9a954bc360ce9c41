run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/fsab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/fsab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2))"
}
run base
MESSI_FILTER_STREAMS=2 run fs2
MESSI_FILTER_STREAMS=2 MESSI_REFINE_STREAMS=4 run fs2_rs4
MESSI_NO_REV=1 run norev
