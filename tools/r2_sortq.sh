mkdir -p gpurun_out
rm -f gpurun_out/sortq.log
timeout 300 python tools/sort_probe.py > gpurun_out/sortq.log 2>&1; echo p=$?
timeout 300 python tools/sort_probe.py --config ads >> gpurun_out/sortq.log 2>&1
timeout 300 python tools/sort_probe.py --alpha 0 >> gpurun_out/sortq.log 2>&1
grep '^{' gpurun_out/sortq.log
timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "dedup or hot_row or small_dense or full_config or multi_step or empty" tests/test_sharded_gpu.py > gpurun_out/sortq_t.log 2>&1; echo t=$?; tail -2 gpurun_out/sortq_t.log
