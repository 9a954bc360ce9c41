# reverse filter v2: DTW stage parity + C4 DTW bench, then ncu of the filter kernel
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dtw_stages or nn_dtw" > gpurun_out/rev2_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/rev2_pytest.log
timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/rev2_bench.log 2>gpurun_out/rev2_bench.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/rev2_bench.log").read().strip().splitlines()[-1])
r = d["roofline"]
print("VALUE", round(d["value"],1), "ms/step", round(d["ms_per_step"],2), "serial", {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()}, "frac", round(r["frac"],3))
print("stats", {k: round(v, 1) for k, v in d["stats_mean"].items()})
PY
MESSI_DTW_REFINE_OCC=1 timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/rev2_bench_occ1.log 2>&1; echo "occ1 rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/rev2_bench_occ1.log").read().strip().splitlines()[-1])
print("OCC1 VALUE", round(d["value"],1), "ms/step", round(d["ms_per_step"],2), "serial", {k: round(v,2) for k,v in d["kernel_ms_per_step"].items()})
PY
bash tools/gpu_ncu_dtw.sh k_lbk_filter_q8r 20 1
python tools/ncu_summary.py gpurun_out/prof_dtw.ncu-rep > gpurun_out/rev2_ncu.txt 2>&1
