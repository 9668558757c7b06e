for a in "--alpha 1.2" "--config jobs" "--config ads" "--alpha 0.8"; do
python bench.py $a --steps 10 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-e2e --no-lib --no-graph | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$a\", d['ms_per_step'], {k:round(v['ms'],4) for k,v in d['phases'].items()})"
done
