# SUSS deferred-search A/B (run under gpurun): parity first, then base vs new on the approx lines
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_approx.py tests/test_gpu_checked.py tests/test_kat_modes.py -q -x > gpurun_out/suss_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/suss_tests.log
for c in 2 5; do
  bash tools/ab.sh "--config $c --approx 10 --steps 5 --warmup 3 --no-e2e --no-cpu" base new base new
done
