# GPU round trip: parity tests, default bench, then one ncu --set full capture of $NCU_RX
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
head -c 600 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
if [ -n "$NCU_RX" ]; then
timeout 300 python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$NCU_RX" -s ${NCU_SKIP:-4} -c ${NCU_COUNT:-1} \
  -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
fi
