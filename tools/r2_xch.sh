mkdir -p gpurun_out
rm -f gpurun_out/xch.jsonl
timeout 1500 python -m pytest -q -x -m gpu tests/test_sharded_gpu.py tests/test_sharded_syncfree_gpu.py tests/test_hostcomm_gpu.py tests/test_feed_model_gpu.py > gpurun_out/xch_t.log 2>&1; echo t=$?; tail -2 gpurun_out/xch_t.log
Q="--steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot"
for a in "--exchange --sharding row" "--exchange --sharding table" "--exchange --sharding row --exchange-mode nccl" "--exchange --sharding table --exchange-mode nccl"; do
  timeout 600 python bench.py $Q $a > gpurun_out/x.log 2>&1
  grep '^{' gpurun_out/x.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args': '$a', 'step_ms': round(d['ms_per_step'],4), 'graph_ms': (d.get('graph') or {}).get('full_ms_per_step_graph'), 'e2e_ms': (d.get('e2e') or {}).get('ms_per_step'), 'phases': {k: [round(v.get('ms',0),4), round(v.get('frac_of_hbm', 0) or 0, 3)] for k, v in d['phases'].items()}}))" | tee -a gpurun_out/xch.jsonl
done
L="--steps 2 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph --no-spot --no-e2e --no-a5 --exchange --sharding row"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/xl2_launches.csv python bench.py $L > gpurun_out/xl2_ncu.log 2>&1; echo l=$?
