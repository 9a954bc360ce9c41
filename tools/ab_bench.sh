# A/B of library builds on the same box: bench.py with MESSI_LIB=<each .so> (C3 ED only)
for lib in "$@"; do
  for rep in 1 2; do
    MESSI_LIB=$lib timeout 600 python bench.py --no-cpu --no-dtw > gpurun_out/ab.log 2>&1
    echo "$lib rep$rep $(grep -o '"value": [0-9.]*' gpurun_out/ab.log | head -1)"
  done
done
