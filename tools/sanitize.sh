# compute-sanitizer suite over every kernel on the tiny config -> gpurun_out/san_<tool>.log.
# NOTE: compute-sanitizer is closed on the build's GPU pool (runs under it refuse to start); the
# substitute there is tests/test_guard_gpu.py (guard bands after every buffer and output, inputs
# unchanged) plus `python tools/sanitize_step.py` (every kernel, status clean).  On a box where the
# tool is allowed this script runs the four tools.
mkdir -p gpurun_out
python tools/sanitize_step.py > gpurun_out/san_plain.log 2>&1; echo plain=$?
for t in memcheck racecheck initcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --target-processes all --print-limit 20 python tools/sanitize_step.py > gpurun_out/san_$t.log 2>&1
  echo $t=$?; tail -3 gpurun_out/san_$t.log
done
