# GPU suite + default bench + serving bench (+ optional extra command); usage: bash tools/r2_check.sh TAG
T=${1:-x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/${T}_tests.log
timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --config feedq8 --steps 20 > gpurun_out/${T}_q8.log 2>&1; echo q8=$?
python - <<PY
import json
for f in ['gpurun_out/${T}_bench.log', 'gpurun_out/${T}_q8.log']:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ph = d.get('phases', {})
        print(f, round(d['ms_per_step'], 4), {k: round(v['ms'], 4) for k, v in ph.items() if isinstance(v, dict) and 'ms' in v}, d['roofline'].get('kernel'), round(d['roofline']['frac'], 3))
    except Exception as e:
        print(f, 'ERR', e)
PY
