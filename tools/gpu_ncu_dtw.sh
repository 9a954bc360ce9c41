# ncu --set full of the DTW refine kernel in the C4 step (one ncu invocation).
# usage: bash tools/gpu_ncu_dtw.sh [regex] [skip] [count] [bench args...]
set -x
RX=${1:-"k_refine_dtw"}; SK=${2:-30}; CN=${3:-1}; shift 3
timeout 300 python bench.py --mode dtw --steps 1 --warmup 3 --queries 20 --no-cpu "$@" > gpurun_out/plain_dtw.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SK -c $CN \
  -o gpurun_out/prof_dtw python bench.py --mode dtw --steps 1 --warmup 3 --queries 20 --no-cpu "$@" > gpurun_out/ncu_dtw.log 2>&1
echo "rc=$?"
