run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/rab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/rab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dtw_stages or nn_dtw" 2>&1 | tail -1
run v4
MESSI_FILTER_STREAMS=2 run v4_fs2
MESSI_AB=1 MESSI_LIB=$PWD/build_variants/libmessi_rb5.so run rb5
MESSI_AB=1 MESSI_LIB=$PWD/build_variants/libmessi_rb5.so MESSI_FILTER_STREAMS=2 run rb5_fs2
