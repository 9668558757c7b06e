mkdir -p gpurun_out
rm -f gpurun_out/sortv.log
for v in 0 1 2 3 4; do
  LIRANK_SORT_VARIANT=$v timeout 300 python tools/sort_probe.py >> gpurun_out/sortv.log 2>&1; echo v$v=$?
  LIRANK_SORT_VARIANT=$v timeout 300 python tools/sort_probe.py --alpha 0 >> gpurun_out/sortv.log 2>&1
done
grep '^{' gpurun_out/sortv.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['variant'], d['alpha'], round(d['sort_ms'],4), round(d['sort_own_frac'],3))"
