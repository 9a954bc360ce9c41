# Round 2 (session 3): the full GPU suite, the default bench line, then a C4 A/B of the reverse
# envelope-PAA filter in the same build (MESSI_NO_RENV=1 turns it off).
set -x
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
for rep in 1; do for v in 1 0; do
  if [ $v = 1 ]; then export MESSI_NO_RENV=1; else unset MESSI_NO_RENV; fi
  timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/bench_dtw_ab.log 2>&1
  python - $v <<'PY'
import json, sys
d = json.loads(open('gpurun_out/bench_dtw_ab.log').read().strip().splitlines()[-1])
sm = d.get('stats_mean', {})
print('NO_RENV=%s' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
      {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
      {k: round(sm.get(k, 0), 1) for k in ('candidates', 'rev_paa_pass', 'lbk_pass', 'refined', 'seed_d2', 'bsf_d2')},
      'lbk frac', round(d['roofline']['lbk_filter']['frac'], 3))
PY
done; done
