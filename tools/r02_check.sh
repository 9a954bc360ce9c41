# GPU tests (all) + the default bench line + the self-launched 2-rank bench
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -rs --durations=12 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -18 gpurun_out/r02_pytest_gpu.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r02_clocks.csv 2>&1 &
SMI=$!
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>gpurun_out/r02_bench.err; echo "bench rc=$?"
kill $SMI
head -c 1500 gpurun_out/r02_bench.log; tail -5 gpurun_out/r02_bench.err
