mkdir -p gpurun_out
Q="--steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot --no-e2e --no-graph"
for v in 0 3 4; do
  for a in 1.05 0; do
    LIRANK_A2_UNR=$v timeout 300 python bench.py $Q --alpha $a > gpurun_out/a2_$v_$a.log 2>&1
    grep '^{' gpurun_out/a2_$v_$a.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('unr', '$v', 'alpha', '$a', 'fwd', round(d['phases']['fwd']['ms'],4), 'step', round(d['ms_per_step'],4))"
  done
done
