# DTW: the w = 64 filter's parity tests, then C4 bench with and without it (MESSI_NO_PAA64)
timeout 1200 python -m pytest -x -q tests/test_gpu_paa64.py tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py ${EXTRA_TESTS} > gpurun_out/dtwtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/dtwtests.log
for rep in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export MESSI_NO_PAA64=1; else unset MESSI_NO_PAA64; fi
  timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/bench_dtw_ab.log 2>&1
  python - $v <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_dtw_ab.log').read().strip().splitlines()[-1])
    sm = d.get('stats_mean', {})
    print('NO_PAA64=%s' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
          {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
          {k: round(sm.get(k, 0)) for k in ('candidates', 'paa_pass', 'lbk_pass', 'refined', 'dtw_cells')})
except Exception as e:
    print('FAILED', e); print(open('gpurun_out/bench_dtw_ab.log').read()[-3000:])
PY
done; done
