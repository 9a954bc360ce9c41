# Round 2 (session 5): the DTW probe pass (MESSI_PROBE = candidates probed before the LB_Keogh
# filters): pruning analysis, C4 A/B over the probe size, DTW suites with the probe on
set -x
timeout 600 python tools/analyze_dtw.py --queries 16 > gpurun_out/analyze_dtw.log 2>&1; echo "analyze rc=$?"; tail -2 gpurun_out/analyze_dtw.log
bash tools/r03_dtw_env.sh - MESSI_PROBE=256 MESSI_PROBE=1024 MESSI_PROBE=2048
MESSI_PROBE=1024 timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py "tests/test_gpu_fullsize.py::test_config4_dtw_10m" > gpurun_out/dtwtests_probe.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dtwtests_probe.log
