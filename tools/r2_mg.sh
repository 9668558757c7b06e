bash tools/r2_bench_n2.sh
bash tools/r2_bench_n4.sh
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/hostcomm_check.py > gpurun_out/hostcomm_torchrun.log 2>&1; echo hc=$?; tail -4 gpurun_out/hostcomm_torchrun.log
