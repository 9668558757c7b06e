# One GPU call: GPU tests, smoke(), the default bench (timed), the reference arm, config/alpha
# variants, the ncu launch list and one ncu --set full capture of a step.  Usage: bash tools/round_check.sh TAG
set -x
T=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? secs=$(( $(date +%s) - start ))
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.log 2>&1; echo ref=$?
Q="--steps 20 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph --no-spot --no-e2e"
timeout 600 python bench.py --alpha 0 $Q > gpurun_out/${T}_cfg_alpha0.log 2>&1; echo a0=$?
timeout 600 python bench.py --config ads $Q > gpurun_out/${T}_cfg_ads.log 2>&1; echo ads=$?
timeout 600 python bench.py --config jobs $Q > gpurun_out/${T}_cfg_jobs.log 2>&1; echo jobs=$?
timeout 900 python bench.py --config feedq8 --steps 20 > gpurun_out/${T}_cfg_feedq8.log 2>&1; echo q8=$?
L="--steps 2 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph --no-spot --no-e2e --no-a5"
timeout 600 python bench.py $L > gpurun_out/ncu_l_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/${T}_launches.csv python bench.py $L > gpurun_out/ncu_l.log 2>&1; echo l=$?
timeout 600 python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ps.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"^k_(pool|radix|onesweep|rle|segreduce|fixup|norm|adagrad|len)" -o gpurun_out/${T}_step_full python tools/profile_step.py --warmup 0 --steps 1 --quantize > gpurun_out/ncu_full.log 2>&1; echo full=$?
# summaries on the box (the copy-back is capped at 64 MiB: a report that would break it stays in /tmp)
python tools/ncu_summary.py gpurun_out/${T}_step_full.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1
for k in k_segreduce k_onesweep k_adagrad_tma k_pool_fwd_f32 k_pool_fwd_q8 k_rle; do
  python tools/ncu_opmix.py gpurun_out/${T}_step_full.ncu-rep "$k" --top 14; echo
done > gpurun_out/${T}_opmix.txt 2>&1
if [ $(stat -c %s gpurun_out/${T}_step_full.ncu-rep) -gt 50000000 ]; then mv gpurun_out/${T}_step_full.ncu-rep /tmp/; echo "rep kept on the box only (size)"; fi
