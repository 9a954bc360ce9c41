for w in 2000 4000 8000 1000; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-dtw --knn 0 --latency 0 --window $w > gpurun_out/w.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/w.log').read().strip().splitlines()[-1]);print('$w',round(d['value']),round(d['stats_mean']['tiles_scanned']),round(d['stats_dist']['bsf0_over_final']['median'],3),{k:round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done
