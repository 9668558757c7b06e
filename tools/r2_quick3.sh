mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_parity.py tests/test_sharded_gpu.py tests/test_serving_gpu.py tests/test_qr_gpu.py tests/test_guard_gpu.py > gpurun_out/q3_t.log 2>&1; echo t=$?; tail -3 gpurun_out/q3_t.log
timeout 600 python bench.py --steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot > gpurun_out/q3_b.log 2>&1; echo b=$?
grep '^{' gpurun_out/q3_b.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4), {k:round(v.get('ms',0),4) for k,v in d['phases'].items()}); print('e2e', d['e2e']['ms_per_step'], 'graph', d.get('graph'))"
timeout 600 python bench.py --alpha 0 --steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot --no-e2e --no-graph > gpurun_out/q3_a0.log 2>&1; echo a0=$?
grep '^{' gpurun_out/q3_a0.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a0 step', round(d['ms_per_step'],4), {k:(round(v.get('ms',0),4), round(v.get('frac_of_hbm',0) or 0,3)) for k,v in d['phases'].items()})"
