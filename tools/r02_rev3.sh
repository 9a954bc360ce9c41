timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py -x -q -k "dtw_stages or nn_dtw or knn" > gpurun_out/rev3_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/rev3_pytest.log
for V in fs1 fs2; do
  if [ $V = fs2 ]; then export MESSI_FILTER_STREAMS=2; fi
  timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/rev3_bench_$V.log 2>gpurun_out/rev3_bench.err; echo "bench rc=$?"
  python - <<PY
import json
d = json.loads(open("gpurun_out/rev3_bench_$V.log").read().strip().splitlines()[-1])
print("$V VALUE", round(d["repeats"]["mean"],1), "ms/step", round(d["ms_per_step"],2), "serial", {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()})
print("stats", {k: round(v, 1) for k, v in d["stats_mean"].items()})
PY
done
unset MESSI_FILTER_STREAMS
bash tools/gpu_ncu_dtw.sh k_lbk_filter_q8r 20 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_dtw.ncu-rep > gpurun_out/rev3_ncu.txt 2>&1
