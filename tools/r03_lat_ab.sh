# C4 DTW single-query latency (p50 / p99) A/B over environment specs (as r03_env_ab.sh).
for spec in "$@"; do
  envs=""
  if [ "$spec" != "-" ]; then envs=$(echo "$spec" | tr ',' ' '); fi
  env $envs timeout 600 python bench.py --mode dtw --steps 2 --warmup 3 --no-cpu --latency 40 --repeats 1 > gpurun_out/bench_lat_ab.log 2>&1
  python - "$spec" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/bench_lat_ab.log').read().strip().splitlines()[-1])
print('ENV=%s' % sys.argv[1], 'value %.1f' % d['value'], 'latency', d.get('latency'))
PY
done
