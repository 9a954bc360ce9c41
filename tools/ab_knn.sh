# A/B of library builds on the k-NN sweep (C2, k = 5, 10, 50), twice each, alternating.
for rep in 1 2; do
for lib in "$@"; do
  MESSI_LIB=$lib timeout 600 python tools/sweep.py --what knn > gpurun_out/abk.jsonl 2>/dev/null
  echo "$lib rep$rep $(python -c "import json;print([(d['k'],round(d['qps'])) for d in map(json.loads,open('gpurun_out/abk.jsonl'))])")"
done
done
