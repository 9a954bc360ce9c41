# A/B of the fused kernel's warps per CTA (build_variants/libmessi_wN.so, -DMESSI_FUSED_WARPS=N)
run() {
  timeout 300 python bench.py --steps 10 --warmup 3 --no-dtw --no-cpu --knn 0 --latency 0 --repeats 3 > gpurun_out/wab.log 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/wab.log').read().strip().splitlines()[-1])
print('$1', round(d['repeats']['mean'],1), round(d['roofline']['frac'],3), d['lib'])"
}
run w12
for W in 11 10; do MESSI_AB=1 MESSI_LIB=$PWD/build_variants/libmessi_w$W.so run w$W; done
