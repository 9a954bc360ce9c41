# usage: bash tools/sanitize.sh memcheck|racecheck|synccheck   (one tool per gpurun call)
TOOL=${1:-memcheck}
EXTRA=""
[ "$TOOL" = "memcheck" ] && EXTRA="--leak-check no"
timeout 240 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"
tail -2 gpurun_out/san_plain.log
timeout 2400 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py \
   > gpurun_out/r02_sanitize_$TOOL.log 2>&1
echo "sanitizer rc=$?"
tail -8 gpurun_out/r02_sanitize_$TOOL.log
