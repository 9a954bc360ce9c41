# A/B of the DTW pipeline shape: refine streams (2 / 4), slots (4 / 8 via build_variants/libmessi_s8.so), refine CTAs per SM
run() {
  timeout 300 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 2 > gpurun_out/dab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/dab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['ms_per_step'],2))"
}
run base
MESSI_REFINE_STREAMS=4 run ref4
export MESSI_AB=1 MESSI_LIB=$PWD/build_variants/libmessi_s8.so
run s8
MESSI_REFINE_STREAMS=4 run s8_ref4
MESSI_REFINE_STREAMS=4 MESSI_DTW_REFINE_OCC=1 run s8_ref4_occ1
MESSI_REFINE_STREAMS=4 MESSI_DTW_REFINE_OCC=2 run s8_ref4_occ2
