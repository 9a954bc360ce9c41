# ncu --set full of the DTW seed and scan kernels (C4 bench), after a plain run exited 0
DARGS="--mode dtw --steps 2 --warmup 3 --no-cpu --latency 0 --repeats 1"
timeout 300 python bench.py $DARGS > gpurun_out/plain_dtw.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_seed_dtw|k_scan\$|k_rev_paa_filter|k_lbk_filter_q8b|k_lbk_rev_q8" -s 100 -c 5 \
  -o gpurun_out/r03_dtw_kernels python bench.py $DARGS > gpurun_out/ncu_dtw.log 2>&1
echo "ncu rc=$?"
