# Round-2 baseline on the GPU: parity tests, default bench line, ncu --set full of the fused ED kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=8 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>gpurun_out/r02_bench.err; echo "bench rc=$?"
head -c 800 gpurun_out/r02_bench.log; tail -3 gpurun_out/r02_bench.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_scan_refine_ed" -s 4 -c 1 \
  -o gpurun_out/r02_fused_base python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
