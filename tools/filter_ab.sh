for F in 0 12 6 3; do
  if [ $F = 0 ]; then unset MESSI_FILTER_CTAS; else export MESSI_FILTER_CTAS=$F; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 3 > gpurun_out/fab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/fab.log').read().strip().splitlines()[-1])
print('F=$F', round(d['repeats']['mean'],1), d['kernel_ms_per_step'])"
done
