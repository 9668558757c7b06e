mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_hostcomm_gpu.py tests/test_gpu_parity.py tests/test_feed_model_gpu.py tests/test_fim_gpu.py tests/test_minmax_gpu.py > gpurun_out/q2_t.log 2>&1; echo t=$?; tail -4 gpurun_out/q2_t.log
timeout 600 python bench.py --steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot > gpurun_out/q2_b.log 2>&1; echo b=$?
grep '^{' gpurun_out/q2_b.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4), {k:round(v.get('ms',0),4) for k,v in d['phases'].items()}); print('e2e', d['e2e']['ms_per_step'], 'graph', d.get('graph'))"
