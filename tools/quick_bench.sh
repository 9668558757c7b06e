mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-e2e > gpurun_out/qb.log 2>&1; echo bench=$?
tail -1 gpurun_out/qb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in d['phases'].items()})"
