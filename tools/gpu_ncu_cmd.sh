# one ncu --set full capture of kernels matching $NCU_RX in the command "$@" (run plain first)
set -x
timeout 600 "$@" > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$NCU_RX" -s ${NCU_SKIP:-4} -c ${NCU_COUNT:-1} \
  -o gpurun_out/prof "$@" > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -c 1500 gpurun_out/plain.log
