# GPU test suite + smoke (one gpurun call)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly "$@" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -30 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
