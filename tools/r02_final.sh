# Round-2 final evidence: the default bench line (what the driver runs), the C3 and C4 launch
# lists, and one ncu --set full capture of the fused ED kernel -- each ncu pass only after the
# same command exited 0 without ncu.
set -x
timeout 1500 python bench.py > gpurun_out/final_bench.log 2> gpurun_out/final_bench.err; echo "bench rc=$?"
ARGS="--steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_c3.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo "launches c3 rc=$?"
DARGS="--mode dtw --steps 2 --warmup 3 --no-cpu --latency 0 --repeats 1"
timeout 300 python bench.py $DARGS > gpurun_out/plain_dtw.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final_launches_c4.csv \
  python bench.py $DARGS > gpurun_out/ncu_launch_dtw.log 2>&1; echo "launches c4 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_scan_refine_ed" -s 4 -c 1 \
  -o gpurun_out/final_fused python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
