mkdir -p gpurun_out
timeout 300 python tools/sort_probe.py --steps 1 > gpurun_out/sp_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_segreduce|k_radix_hist" -s 15 -c 5 -o gpurun_out/sort_full python tools/sort_probe.py --steps 1 > gpurun_out/ncu_sort.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_sort.log
