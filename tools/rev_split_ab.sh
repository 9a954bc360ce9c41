run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/rsab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/rsab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, 'lbk_pass', round(d['stats_mean']['lbk_pass']), 'cells', round(d['stats_mean']['dtw_cells']/1e6))"
}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py -x -q -k "dtw_stages or nn_dtw or knn" 2>&1 | tail -2
run split1
MESSI_REV_RHO=0.7 run split07
MESSI_REV_RHO=0.5 run split05
MESSI_REV_RHO=0.3 run split03
MESSI_REV_MODE=fused run fused
