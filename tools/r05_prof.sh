# Round 2 (session 5): launch lists at HEAD (C3 and C4; ncu per-launch device times are cold
# and serialised -- shares, not absolutes) and one ncu --set full pass over the DTW stage
# kernels of one mid-run C4 query; each ncu pass only after the same command exited 0 plain.
set -x
ARGS="--steps 2 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 1"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r05_launches_c3.csv \
  python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo "launches c3 rc=$?"
DARGS="--mode dtw --steps 1 --warmup 3 --no-cpu --latency 0 --repeats 1"
timeout 300 python bench.py $DARGS > gpurun_out/plain_dtw.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4500 --csv --log-file gpurun_out/r05_launches_c4.csv \
  python bench.py $DARGS > gpurun_out/ncu_launch_dtw.log 2>&1; echo "launches c4 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_rev_paa_filter|k_lbk_filter_q8b|k_lbk_rev_q8|k_refine_dtw_strip" -s 240 -c 4 \
  -o gpurun_out/r05_dtw_full python bench.py $DARGS > gpurun_out/ncu_full_dtw.log 2>&1
echo "ncu rc=$?"
