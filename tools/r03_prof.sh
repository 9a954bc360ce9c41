# Launch list (device time of every launch) and one ncu --set full capture of the fused ED
# kernel for the C3 bench, each after the same command exited 0 without ncu.
set -x
ARGS="--steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${NCU_OUT:-r03}_launches.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K:-k_scan_refine_ed}" -s 4 -c 1 \
  -o gpurun_out/${NCU_OUT:-r03}_full python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
