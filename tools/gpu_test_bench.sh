# GPU parity tests + default bench (+ optional extra bench args in $BENCH_ARGS)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log; tail -5 gpurun_out/bench.err
