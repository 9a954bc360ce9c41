run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 --steady 0 > gpurun_out/tab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/tab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dtw_stages or nn_dtw" 2>&1 | tail -1
export MESSI_AB=1
MESSI_LIB=$PWD/build_variants/libmessi_head.so run head
MESSI_LIB=$PWD/build_variants/libmessi_tail.so run tail
MESSI_LIB=$PWD/build_variants/libmessi_head.so run head2
MESSI_LIB=$PWD/build_variants/libmessi_tail.so run tail2
