# DTW C4 bench under several environment settings (each argument: "VAR=val VAR2=val" or "-")
for rep in 1 2; do for envs in "$@"; do
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/bench_dtw_env.log 2>&1
  python - "$envs" <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_dtw_env.log').read().strip().splitlines()[-1])
    sm = d.get('stats_mean', {})
    print('ENV[%s]' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
          {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
          {k: round(sm.get(k, 0)) for k in ('candidates', 'paa_pass', 'reverse_evaluated', 'lbk_pass', 'refined')})
except Exception as e:
    print('FAILED', e); print(open('gpurun_out/bench_dtw_env.log').read()[-3000:])
PY
done; done
