run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/k2ab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/k2ab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
}
export MESSI_AB=1
MESSI_LIB=$PWD/build_variants/libmessi_nopf.so run nopf
MESSI_LIB=$PWD/build_variants/libmessi_pf.so run pf
