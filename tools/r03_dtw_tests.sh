# The DTW parity / k-NN / shard suites and the full-size C4 test, then EXTRA (a command).
timeout 1800 python -m pytest -q -rs tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py "tests/test_gpu_fullsize.py::test_config4_dtw_10m" > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dtwtests.log
