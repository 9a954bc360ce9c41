# A/B of library builds on the same box, alternating (A B A B ...): bench.py C3 ED with
# MESSI_LIB=<each .so>, value / roofline frac / fused-kernel ms per step.  Usage: ab_alt.sh REPS a.so b.so ...
reps=$1; shift
for rep in $(seq 1 $reps); do
  for lib in "$@"; do
    MESSI_AB=1 MESSI_LIB=$lib timeout 600 python bench.py --no-cpu --no-dtw --knn 0 --latency 0 --repeats 3 ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
    python - "$lib" "$rep" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1])
    print("AB", sys.argv[1], "rep", sys.argv[2], "value %.0f" % d["value"], "mean %.0f" % d["repeats"]["mean"],
          "frac %.4f" % d["roofline"]["frac"], "scan_ms %.4f" % d["kernel_ms_per_step"]["scan"], "pre_ms %.4f" % d["kernel_ms_per_step"]["seed"], "ms/step %.4f" % d["ms_per_step"],
          "traffic", d["roofline"].get("traffic"), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print("AB", sys.argv[1], "FAILED", e); print(open("gpurun_out/ab.log").read()[-2000:])
PY
  done
done
