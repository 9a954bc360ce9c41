# DTW parity + the C4 DTW bench line (serial per-kernel breakdown included)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -rs -k "dtw or distances" > gpurun_out/dtw_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/dtw_pytest.log
timeout 600 python bench.py --mode dtw --steps 2 --warmup 1 --no-cpu --latency 0 --repeats 1 > gpurun_out/dtw_bench.log 2>gpurun_out/dtw_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/dtw_bench.log").read().strip().splitlines()[-1])
r = d["roofline"]
print("VALUE", d["value"], "ms/step", d["ms_per_step"], "serial", d["kernel_ms_per_step"], "frac", r["frac"], "lbk", r["lbk_filter"])
print("stats", {k: round(v, 1) for k, v in d["stats_mean"].items()})
PY
tail -3 gpurun_out/dtw_bench.err
