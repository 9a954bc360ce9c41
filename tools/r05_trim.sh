# Round 2 (session 5): short-list CTA trimming of the strip refine: C4 A/B (MESSI_DTW_TRIM=0: off), then the DTW suites
bash tools/r03_dtw_env.sh - MESSI_DTW_TRIM=0
bash tools/r03_dtw_env.sh - MESSI_DTW_TRIM=0
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py "tests/test_gpu_fullsize.py::test_config4_dtw_10m" > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dtwtests.log
timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 20 --repeats 3 > gpurun_out/bench_dtw.log 2>&1; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_dtw.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['repeats']['qps'], d['roofline']['steady_state']['frac'], d['roofline']['frac'], d.get('latency'))"
