run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/bab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/bab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, 'lbk_pass', round(d['stats_mean']['lbk_pass']))"
}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py -x -q -k "dtw_stages or nn_dtw or knn" 2>&1 | tail -2
run bulk
MESSI_LBK_BULK=0 run ldg
bash tools/gpu_ncu_dtw.sh k_lbk_rev_q8 20 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_dtw.ncu-rep > gpurun_out/bulk_ncu.txt 2>&1
