mkdir -p gpurun_out

grep '"rank"' gpurun_out/hostcomm_torchrun.log | cut -c1-200
timeout 300 python tools/sort_probe.py --steps 1 > gpurun_out/sp_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_segreduce|k_pool_fwd_f32|k_adagrad" -s 9 -c 3 -o gpurun_out/r02_v3_kern python tools/sort_probe.py --steps 1 > gpurun_out/ncu_v3.log 2>&1; echo ncu=$?
