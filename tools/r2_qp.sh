mkdir -p gpurun_out
Q="--steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph --no-spot --no-e2e --no-a5"
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export LIRANK_QPITCH64=1; else unset LIRANK_QPITCH64; fi
  timeout 600 python bench.py $Q > gpurun_out/qp_f_$v.log 2>&1
  timeout 600 python bench.py $Q --alpha 0 > gpurun_out/qp_a_$v.log 2>&1
  timeout 900 python bench.py --config feedq8 --steps 20 > gpurun_out/qp_s_$v.log 2>&1
  python - <<PY
import json
for n in ['f','a','s']:
    d=json.loads(open('gpurun_out/qp_%s_$v.log' % n).read().strip().splitlines()[-1])
    ph=d.get('phases',{})
    print('v=$v', n, round(d['ms_per_step'],4), 'a8', round(ph.get('update',{}).get('ms',0),4), 'a10', round(ph.get('fwd_q8',{}).get('ms',0),4), d['config'].get('q8_store_bytes'))
PY
done
unset LIRANK_QPITCH64
LIRANK_QPITCH64=1 timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_minmax_gpu.py tests/test_serving_gpu.py > gpurun_out/qp_t.log 2>&1; echo t=$?; tail -1 gpurun_out/qp_t.log
