# default bench (N=1) + reference arm + exchange-path bench + a new test file (one gpurun call)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -c 800 gpurun_out/bench_ref.log
timeout 600 python bench.py --exchange --steps 10 --no-cpu --no-qr --no-model --no-fim --no-lib > gpurun_out/bench_exch.log 2>&1; echo exch=$?
timeout 900 python -m pytest -q tests/test_gpu_parity.py tests/test_feed_model_gpu.py > gpurun_out/t.log 2>&1; echo t=$?; tail -3 gpurun_out/t.log
