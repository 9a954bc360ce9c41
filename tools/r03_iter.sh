# Iteration: parity suites for the ED path, then one ncu --set full capture of the fused kernel (C3)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn.py tests/test_gpu_shards.py tests/test_gpu_tc.py -x -q -rs > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/it_pytest.log
ARGS="--steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_scan_refine_ed" -s 4 -c 1 \
  -o gpurun_out/${NCU_OUT:-r03_fused} python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
