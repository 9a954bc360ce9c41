# The checked build (bounds asserts, MESSI_CHECKED) run through the parity / k-NN / TC tests and
# the all-paths sanitize run: an out-of-capacity index traps the kernel and fails the run.
set -x
export MESSI_LIB=$PWD/paper_2110_07519_b200/libmessi_checked.so
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn.py tests/test_gpu_knn_dtw.py tests/test_gpu_tc.py \
    tests/test_gpu_shards.py -x -q -rs > gpurun_out/${TAG:-r02}_checked_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG:-r02}_checked_pytest.log
timeout 600 python tools/sanitize_run.py > gpurun_out/${TAG:-r02}_checked_run.log 2>&1; echo "run rc=$?"
tail -3 gpurun_out/${TAG:-r02}_checked_run.log
