# Quick iteration: parity tests (no full-size), then a short C3 bench line
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_knn.py tests/test_gpu_shards.py -x -q -rs > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/it_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-dtw --no-cpu --knn 10 --latency 10 --repeats 3 ${BENCH_ARGS} > gpurun_out/it_bench.log 2>gpurun_out/it_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/it_bench.log").read().strip().splitlines()[-1])
print("VALUE", d["value"], "frac", d["roofline"]["frac"], "kernel_ms", d["kernel_ms_per_step"], "knn", d.get("knn", {}).get("value"),
      "repeats", d["repeats"]["mean"], "lat", d.get("latency", {}).get("p50_ms"))
print("stats", {k: round(v, 1) for k, v in d["stats_mean"].items()})
PY
tail -3 gpurun_out/it_bench.err
