# One GPU call: GPU tests, smoke(), the default bench (timed), launch list + ncu full capture.
set -x
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
start=$(date +%s); python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$? secs=$(( $(date +%s) - start ))
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph > gpurun_out/ncu_l.log 2>&1; echo l=$?
python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ps.log 2>&1; echo ps=$?
ncu --set full --clock-control none --import-source on -k regex:"^k_(pool|radix|onesweep|rle|segreduce|fixup|norm|adagrad|quantize|len)" -o gpurun_out/step_full python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ncu_full.log 2>&1; echo full=$?
