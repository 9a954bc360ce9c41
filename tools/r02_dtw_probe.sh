timeout 600 python tools/analyze_lb_rev.py --queries 6 > gpurun_out/lbrev_h8.log 2>&1; echo "a rc=$?"
timeout 300 python tools/analyze_lb_rev.py --queries 3 --H 4 > gpurun_out/lbrev_h4.log 2>&1; echo "b rc=$?"
bash tools/gpu_ncu_dtw.sh k_refine_dtw_strip 30 1
ncu -i gpurun_out/prof_dtw.ncu-rep --page raw --csv > gpurun_out/prof_dtw_raw.csv 2>/dev/null
python tools/ncu_sass_mix.py gpurun_out/prof_dtw.ncu-rep 30 > gpurun_out/prof_dtw_sass.txt 2>&1
