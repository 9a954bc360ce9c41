# Reverse LB_Keogh filter: DTW parity + end-to-end DTW tests, then the C4 DTW bench with and without it
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py tests/test_gpu_fullsize.py -x -q -k "dtw or distances or knn or c4" > gpurun_out/rev_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/rev_pytest.log
for V in rev norev; do
  if [ $V = norev ]; then export MESSI_NO_REV=1; fi
  timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/rev_bench_$V.log 2>gpurun_out/rev_bench_$V.err; echo "bench $V rc=$?"
  python - <<PY
import json
d = json.loads(open("gpurun_out/rev_bench_$V.log").read().strip().splitlines()[-1])
r = d["roofline"]
print("$V VALUE", round(d["value"],1), "ms/step", round(d["ms_per_step"],2), "serial", {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()}, "frac", round(r["frac"],3), "lbk", r.get("lbk_filter"))
print("stats", {k: round(v, 1) for k, v in d["stats_mean"].items()})
PY
done
