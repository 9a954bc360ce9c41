# ED C3 bench under several environment settings (each argument: "VAR=val" or "-"), alternated
for rep in 1 2; do for envs in "$@"; do
  [ "$envs" = "-" ] && envs=""
  env $envs timeout 600 python bench.py --no-dtw --no-cpu --knn 0 --latency 0 --repeats 3 > gpurun_out/bench_ed_env.log 2>/dev/null
  python - "$envs" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/bench_ed_env.log').read().strip().splitlines()[-1])
print('ENV[%s]' % sys.argv[1], [round(x) for x in d['repeats']['qps']], {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if v})
PY
done; done
