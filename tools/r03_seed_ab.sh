# DTW selective seed: DTW parity suites, then C4 bench A/B alternating MESSI_SEED_M=0 (every
# window row) and the default (32 best LB_Keogh-ranked rows); EXTRA_M adds more M values.
timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_knn_dtw.py -k "dtw or DTW" > gpurun_out/seedtests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/seedtests.log
for rep in 1 2; do for m in 0 default ${EXTRA_M}; do
  if [ $m = default ]; then unset MESSI_SEED_M; else export MESSI_SEED_M=$m; fi
  timeout 600 python bench.py --mode dtw --steps 3 --warmup 3 --no-cpu --latency 0 --repeats 1 > gpurun_out/bench_dtw_ab.log 2>&1
  python - $m <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/bench_dtw_ab.log').read().strip().splitlines()[-1])
    sm = d.get('stats_mean', {})
    print('SEED_M=%s' % sys.argv[1], 'value %.1f' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
          {k: round(v, 2) for k, v in d.get('kernel_ms_per_step_serial', d.get('kernel_ms_per_step', {})).items()},
          {k: round(sm.get(k, 0), 3) for k in ('candidates', 'lbk_pass', 'refined', 'dtw_cells', 'seed_d2', 'bsf_d2')})
except Exception as e:
    print('FAILED', e); print(open('gpurun_out/bench_dtw_ab.log').read()[-3000:])
PY
done; done
# one ncu --set full capture of the DTW scan (k_scan) after the plain run above exited 0
DARGS="--mode dtw --steps 2 --warmup 3 --no-cpu --latency 0 --repeats 1"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_scan\$" -s 20 -c 1 \
  -o gpurun_out/r03_scan_dtw python bench.py $DARGS > gpurun_out/ncu_scan.log 2>&1; echo "ncu rc=$?"
