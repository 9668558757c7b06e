mkdir -p gpurun_out
rm -f gpurun_out/sortq.log
timeout 300 python tools/sort_probe.py > gpurun_out/sortq.log 2>&1; echo p=$?
timeout 300 python tools/sort_probe.py --config ads >> gpurun_out/sortq.log 2>&1
timeout 300 python tools/sort_probe.py --alpha 0 >> gpurun_out/sortq.log 2>&1
grep '^{' gpurun_out/sortq.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['alpha'], 'sort', round(d['sort_ms'],4), 'rle', round(d['rle_ms'],4), 'a5 own frac', round(d['a5_own_frac'],3))"
timeout 1200 python -m pytest -q tests/test_gpu_parity.py tests/test_sharded_gpu.py tests/test_sharded_syncfree_gpu.py tests/test_graph_gpu.py > gpurun_out/sortq_t.log 2>&1; echo t=$?; tail -2 gpurun_out/sortq_t.log
