# One GPU call: the default bench, then the ncu launch list of a short bench run and a
# --set full capture of one step's kernels (tools/profile_step.py).  Outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_s2.log 2>&1; echo b2=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_l.log 2>&1; echo l=$?
python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ps.log 2>&1; echo ps=$?
ncu --set full --clock-control none --import-source on -k regex:"^k_(pool|radix|onesweep|rle|segreduce|fixup|norm|adagrad|quantize)" -o gpurun_out/step_full python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ncu_full.log 2>&1; echo full=$?
