# the whole GPU suite (with durations) and smoke
set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
