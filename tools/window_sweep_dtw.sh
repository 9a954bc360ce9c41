for w in 2000 4000 1000; do
timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --window $w > gpurun_out/w.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/w.log').read().strip().splitlines()[-1]);s=d['stats_mean'];print('$w',round(d['value']),round(s['candidates']),round(s['lbk_pass']),round(d['stats_dist']['bsf0_over_final']['median'],3),{k:round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
done
