# slab tests (split halves), the multi-GPU test (skips on one GPU), then compute-sanitizer memcheck on
# tools/sanitize_run.py after a plain run of the same command
set -x
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_slab_ipc.py tests/test_gpu_multi.py -x -q > gpurun_out/pytest_slab.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/pytest_slab.log
timeout 600 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1800 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_memcheck.log 2>&1; echo memcheck_rc=$?
tail -8 gpurun_out/sanitize_memcheck.log
