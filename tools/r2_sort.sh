mkdir -p gpurun_out
for v in 0 1 2 3; do
  LIRANK_SORT_VARIANT=$v timeout 300 python tools/sort_probe.py >> gpurun_out/sort_probe.log 2>&1; echo v$v=$?
  LIRANK_SORT_VARIANT=$v timeout 300 python tools/sort_probe.py --config ads >> gpurun_out/sort_probe.log 2>&1
done
for v in 1 2; do
LIRANK_SORT_VARIANT=$v timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "dedup or hot_row or small_dense or full_config" > gpurun_out/sort_t$v.log 2>&1; echo t$v=$?; tail -2 gpurun_out/sort_t$v.log
done
grep '^{' gpurun_out/sort_probe.log
