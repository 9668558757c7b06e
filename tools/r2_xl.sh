# ncu launch list of the 1-rank sharded (fused, row-wise) step: per-kernel times of the exchange path
mkdir -p gpurun_out
L="--steps 2 --warmup 3 --no-cpu --no-qr --no-model --no-fim --no-lib --no-graph --no-spot --no-e2e --no-a5 --exchange --sharding row"
timeout 600 python bench.py $L > gpurun_out/xl_plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/xl_launches.csv python bench.py $L > gpurun_out/xl_ncu.log 2>&1; echo l=$?
