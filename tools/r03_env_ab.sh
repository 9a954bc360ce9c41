# C4 A/B over environment settings of the same build: each argument is a space-free list of
# VAR=value pairs joined by commas ("-" = none).  Usage: r03_env_ab.sh REPS spec1 spec2 ...
reps=$1; shift
for rep in $(seq 1 $reps); do for spec in "$@"; do
  envs=""
  if [ "$spec" != "-" ]; then envs=$(echo "$spec" | tr ',' ' '); fi
  env $envs timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 ${BENCH_ARGS} > gpurun_out/bench_env_ab.log 2>&1
  python - "$spec" <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_env_ab.log').read().strip().splitlines()[-1])
    sm = d.get('stats_mean', {})
    print('ENV=%s' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
          {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
          {k: round(sm.get(k, 0), 1) for k in ('candidates', 'rev_paa_pass', 'lbk_pass', 'refined', 'dtw_cells', 'seed_d2')})
except Exception as e:
    print('ENV=%s FAILED' % sys.argv[1], e); print(open('gpurun_out/bench_env_ab.log').read()[-2000:])
PY
done; done
