# DTW A/B of library builds on one box, alternating: C4 bench with MESSI_LIB=<each .so>.
# Usage: r03_dtw_lib_ab.sh REPS a.so b.so ...   (TESTS=1: the DTW parity suites first, in-tree lib)
reps=$1; shift
if [ -n "$TESTS" ]; then
timeout 1500 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py tests/test_gpu_shards.py ${EXTRA_TESTS} > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dtwtests.log
fi
for rep in $(seq 1 $reps); do for lib in "$@"; do
  MESSI_AB=1 MESSI_LIB=$lib timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/bench_dtw_ab.log 2>&1
  python - $lib <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_dtw_ab.log').read().strip().splitlines()[-1])
    sm = d.get('stats_mean', {})
    print('LIB=%s' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
          {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
          {k: round(sm.get(k, 0), 3) for k in ('candidates', 'lbk_pass', 'refined', 'dtw_cells', 'seed_d2', 'bsf_d2')})
except Exception as e:
    print('FAILED', e); print(open('gpurun_out/bench_dtw_ab.log').read()[-3000:])
PY
done; done
