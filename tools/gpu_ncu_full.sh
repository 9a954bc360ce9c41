# ncu --set full of the top kernels of the C3 ED step (one ncu invocation).
# usage: bash tools/gpu_ncu_full.sh <regex> <skip> <count> [bench args...]
set -x
RX=${1:-"k_scan|k_refine_ed"}; SK=${2:-40}; CN=${3:-4}; shift 3
timeout 300 python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu "$@" > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s $SK -c $CN \
  -o gpurun_out/prof python bench.py --steps 2 --warmup 3 --no-dtw --no-cpu "$@" > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
