# DTW parity tests + C4 bench (A/B via MESSI_LIB when arguments are given).
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py -m gpu -k "dtw" > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/dtwtests.log
for rep in 1 2; do for lib in "$@"; do
MESSI_LIB=$lib timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_dtw_ab.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_dtw_ab.log').read().strip().splitlines()[-1]);print('$lib',d['value'],round(d['roofline']['frac'],3),{k:round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
done; done
