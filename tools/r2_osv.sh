mkdir -p gpurun_out
rm -f gpurun_out/osv.log
for v in 0 1 2 3 4; do
  LIRANK_OS_VARIANT=$v timeout 300 python tools/sort_probe.py >> gpurun_out/osv.log 2>&1; echo v$v=$?
  LIRANK_OS_VARIANT=$v timeout 300 python tools/sort_probe.py --config ads >> gpurun_out/osv.log 2>&1
done
grep '^{' gpurun_out/osv.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['variant'] if 'variant' in d else '', round(d['sort_ms'],4), round(d['sort_own_frac'],3))"
for v in 1 2; do
LIRANK_OS_VARIANT=$v timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "dedup or hot_row or full_config or small_dense or empty" > gpurun_out/osv_t$v.log 2>&1; echo t$v=$?; tail -1 gpurun_out/osv_t$v.log
done
