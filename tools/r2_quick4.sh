mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_parity.py tests/test_minmax_gpu.py tests/test_serving_gpu.py tests/test_sharded_gpu.py -k "q8 or minmax or serving or full_config or quantize" > gpurun_out/q4_t.log 2>&1; echo t=$?; tail -3 gpurun_out/q4_t.log
timeout 600 python bench.py --steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot > gpurun_out/q4_b.log 2>&1; echo b=$?
grep '^{' gpurun_out/q4_b.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4), {k:round(v.get('ms',0),4) for k,v in d['phases'].items()}); print('e2e', d['e2e']['ms_per_step'], 'graph', d.get('graph'))"
timeout 600 python bench.py --alpha 0 --steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot --no-e2e --no-graph > gpurun_out/q4_a0.log 2>&1; echo a0=$?
grep '^{' gpurun_out/q4_a0.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a0 step', round(d['ms_per_step'],4), {k:(round(v.get('ms',0),4), round(v.get('frac_of_hbm',0) or 0,3)) for k,v in d['phases'].items()})"
timeout 600 python bench.py --config feedq8 --steps 20 --no-cpu > gpurun_out/q4_q8.log 2>&1; echo q8=$?
grep '^{' gpurun_out/q4_q8.log | tail -1 | cut -c1-400
