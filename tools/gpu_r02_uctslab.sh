set -x
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_uct.py tests/test_gpu_slab_ipc.py -x -q > gpurun_out/pytest_uctslab.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_uctslab.log
