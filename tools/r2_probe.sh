# quick A/B probe: a5/a6/a8 phase times alone (tools/sort_probe.py), twice each, then the parity suites
mkdir -p gpurun_out
rm -f gpurun_out/probe.log
for r in 1 2; do
  timeout 300 python tools/sort_probe.py >> gpurun_out/probe.log 2>&1; echo f$r=$?
  timeout 300 python tools/sort_probe.py --config ads >> gpurun_out/probe.log 2>&1
  timeout 300 python tools/sort_probe.py --alpha 0 >> gpurun_out/probe.log 2>&1
done
grep '^{' gpurun_out/probe.log | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['alpha'], 'sort', round(d['sort_ms'],4), 'rle', round(d['rle_ms'],4), 'a6', round(d['segreduce_ms'],4), 'a8', round(d['update_ms'],4))"
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_feed_model_gpu.py tests/test_sharded_syncfree_gpu.py tests/test_sharded_gpu.py tests/test_graph_gpu.py > gpurun_out/probe_t.log 2>&1; echo t=$?; tail -2 gpurun_out/probe_t.log
