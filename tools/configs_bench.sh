# One GPU call: the other BASELINE configs and the alpha sensitivity at N = 1 (bench lines -> gpurun_out/cfg_*.json)
mkdir -p gpurun_out
for c in jobs jobs_shared ads; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-qr --no-model --no-fim > gpurun_out/cfg_$c.log 2>&1; echo $c=$?
  tail -1 gpurun_out/cfg_$c.log > gpurun_out/cfg_$c.json
done
for a in 0 0.8 1.2; do
  timeout 400 python bench.py --alpha $a --steps 10 --warmup 3 --no-cpu --no-qr --no-model --no-fim > gpurun_out/cfg_alpha$a.log 2>&1; echo alpha$a=$?
  tail -1 gpurun_out/cfg_alpha$a.log > gpurun_out/cfg_alpha$a.json
done
timeout 900 python bench.py --config feedq8 --steps 10 --warmup 3 > gpurun_out/cfg_feedq8.log 2>&1; echo feedq8=$?
tail -1 gpurun_out/cfg_feedq8.log > gpurun_out/cfg_feedq8.json
