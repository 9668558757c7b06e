# Quick Feed-1 bench (no CPU baseline / QR / model / FIM sections): step time + per-phase ms
mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-qr --no-model --no-fim "$@" > gpurun_out/qb.log 2>&1; echo bench=$?
tail -1 gpurun_out/qb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in d['phases'].items()}); print('graph', d.get('graph')); print('lib', d.get('library')); print('e2e', d.get('e2e'))"
