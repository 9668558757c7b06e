mkdir -p gpurun_out
for c in ads jobs; do
timeout 1500 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --transport host --config $c --steps 2 --warmup 2 --no-e2e > gpurun_out/bench_n4_$c.log 2>&1; echo n4$c=$?
grep '^{' gpurun_out/bench_n4_$c.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({k: d[k] for k in ('value','ms_per_step','n_gpus','scaling','spot_check','per_rank_ms') if k in d})[:1500])"
done
