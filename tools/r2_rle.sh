mkdir -p gpurun_out
rm -f gpurun_out/rle.log
for v in 16 8 24 32; do
  LIRANK_RLE_ITEMS=$v timeout 300 python tools/sort_probe.py >> gpurun_out/rle.log 2>&1; echo v$v=$?
done
grep '^{' gpurun_out/rle.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(round(d['sort_ms'],4), round(d['rle_ms'],4))"
LIRANK_RLE_ITEMS=32 timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "dedup or hot_row or full_config or small_dense or empty" > gpurun_out/rle_t.log 2>&1; echo t=$?; tail -2 gpurun_out/rle_t.log
