# final pass of this session (run under gpurun): the default bench line, then the full GPU suite
set -u
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/r02h_default.json 2> gpurun_out/r02h_default.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r02h_default.json
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02h_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02h_gpu_tests.log
