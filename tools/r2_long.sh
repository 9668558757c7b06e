# steady-state check: the default bench three times, then one 300-step run (clocks sampled throughout)
mkdir -p gpurun_out
for r in 1 2 3; do timeout 600 python bench.py --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot > gpurun_out/long_$r.log 2>&1; echo r$r=$?; done
timeout 900 python bench.py --steps 300 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot --no-graph > gpurun_out/long_300.log 2>&1; echo r300=$?
for f in gpurun_out/long_1.log gpurun_out/long_2.log gpurun_out/long_3.log gpurun_out/long_300.log; do
  tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['steps'], round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), d['clocks'])"
done
