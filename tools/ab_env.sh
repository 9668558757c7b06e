# A/B a temporary environment knob on the Feed-1 step: bash tools/ab_env.sh VAR "v1 v2 ..." [bench args]
VAR=$1; VALS=$2; shift 2
mkdir -p gpurun_out
Q="--steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-spot --no-e2e --no-graph"
for v in $VALS; do
  for a in 1.05 0; do
    env $VAR=$v timeout 300 python bench.py $Q --alpha $a "$@" > gpurun_out/ab_${v}_$a.log 2>&1
    grep '^{' gpurun_out/ab_${v}_$a.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR', '$v', 'alpha', '$a', 'step', round(d['ms_per_step'],4), {k: round(v['ms'],4) for k, v in d['phases'].items() if k in ('fwd','segreduce','update','fwd_q8','a5_dedup')})"
  done
done
