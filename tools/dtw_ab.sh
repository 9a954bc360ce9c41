# C4 bench A/B of DTW refine occupancy (strip kernel), plus one serial run for the stage breakdown.
for cfg in "1 0" "1 4" "1 3"; do set -- $cfg
MESSI_DTW_STRIP=$1 MESSI_DTW_REFINE_OCC=$2 timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_dtw_o$2.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_dtw_o$2.log').read().strip().splitlines()[-1]);print('occ=$2',d['value'],d['roofline']['frac'],{k:round(v,1) for k,v in d['kernel_ms_per_step'].items()},d['stats_mean']['dtw_cells'])"
done
MESSI_SERIAL=1 MESSI_DTW_STRIP=1 timeout 300 python bench.py --mode dtw --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_dtw_ser.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_dtw_ser.log').read().strip().splitlines()[-1]);print('serial',d['value'],d['roofline']['frac'],{k:round(v,1) for k,v in d['kernel_ms_per_step'].items()},d['stats_mean']['dtw_cells'])"
