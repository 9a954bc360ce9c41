# ncu summaries for profiles/: tensor-core kernel (C2, 100 and 256 queries), DTW filters and refine (C4), DTW launch list
set -x
timeout 300 python tools/tc_ncu.py 100 > gpurun_out/p2_tc_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ed_tc -s 2 -c 1 -o gpurun_out/p2_tc100 python tools/tc_ncu.py 100 > gpurun_out/p2_tc_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ed_tc -s 2 -c 1 -o gpurun_out/p2_tc256 python tools/tc_ncu.py 256 >> gpurun_out/p2_tc_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p2_tc100.ncu-rep > gpurun_out/p2_tc_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/p2_tc256.ncu-rep >> gpurun_out/p2_tc_summary.txt 2>&1
timeout 300 python bench.py --mode dtw --steps 1 --warmup 3 --queries 20 --no-cpu --steady 0 > gpurun_out/p2_dtw_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_lbk_filter_q8b|k_lbk_rev_q8|k_refine_dtw_strip" -s 60 -c 3 -o gpurun_out/p2_dtw python bench.py --mode dtw --steps 1 --warmup 3 --queries 20 --no-cpu --steady 0 > gpurun_out/p2_dtw_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p2_dtw.ncu-rep > gpurun_out/p2_dtw_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p2_launches_c4.csv python bench.py --mode dtw --steps 1 --warmup 1 --queries 20 --no-cpu --steady 0 --latency 0 --repeats 1 > gpurun_out/p2_launch.log 2>&1
echo done
python tools/ncu_sass_mix.py gpurun_out/p2_dtw.ncu-rep 8 > gpurun_out/p2_dtw_sass.txt 2>&1
python tools/ncu_sass_mix.py gpurun_out/p2_tc256.ncu-rep 8 > gpurun_out/p2_tc_sass.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
