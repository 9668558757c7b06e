# selected GPU tests + quick Feed-1 bench (one gpurun call)
mkdir -p gpurun_out
timeout 1500 python -m pytest -q "$@" > gpurun_out/gpu_tests_q.log 2>&1; echo tests=$?
tail -8 gpurun_out/gpu_tests_q.log
bash tools/quick_bench.sh
