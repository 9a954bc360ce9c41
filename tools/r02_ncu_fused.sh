# DTW k-NN + parity tests, then one ncu --set full capture of the fused ED kernel (C3 bench)
set -x
timeout 900 python -m pytest tests/test_gpu_knn_dtw.py tests/test_gpu_parity.py tests/test_gpu_knn.py -x -q -rs > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/it_pytest.log
ARGS="--steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_scan_refine_ed" -s 4 -c 1 \
  -o gpurun_out/${NCU_OUT:-r02_fused} python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
