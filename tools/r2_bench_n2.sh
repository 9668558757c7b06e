# the N=2 bench path (strong-scaling plan, in-run spot check, per-rank times, e2e) with both ranks
# on this one GPU through the host transport (functional check; not NVLink timing)
mkdir -p gpurun_out
timeout 1500 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --transport host --steps 3 --warmup 2 > gpurun_out/bench_n2_host.log 2>&1; echo n2=$?
grep '^{' gpurun_out/bench_n2_host.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({k: d[k] for k in ('value','ms_per_step','n_gpus','scaling','config','spot_check','per_rank_ms','e2e') if k in d})[:3000])"
tail -5 gpurun_out/bench_n2_host.log | cut -c1-300
timeout 1500 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --transport host --config ads --steps 2 --warmup 2 --no-e2e > gpurun_out/bench_n2_ads.log 2>&1; echo n2ads=$?
grep '^{' gpurun_out/bench_n2_ads.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({k: d[k] for k in ('value','ms_per_step','n_gpus','scaling','spot_check','per_rank_ms') if k in d})[:2000])"
