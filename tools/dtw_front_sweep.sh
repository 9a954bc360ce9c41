for f in 0.5 0.3 0.7 0; do
MESSI_DTW_FRONT=$f timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 > gpurun_out/f.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/f.log').read().strip().splitlines()[-1]);print('$f',round(d['value']),round(d['stats_mean']['dtw_cells']/1e6),{k:round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
done
