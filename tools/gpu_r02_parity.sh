set -x
nproc; free -g; lscpu | grep -i "model name\|^CPU(s)\|Thread\|Socket"
export ECHO_PARITY_LOG=$PWD/gpurun_out/parity_scales.jsonl
rm -f $ECHO_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu.log
ECHO_FULL_CFG3=1 timeout 1800 python -m pytest tests/test_gpu_fullsize.py -k cfg3 -q -s > gpurun_out/fullsize_cfg3.log 2>&1; echo cfg3_rc=$?
tail -5 gpurun_out/fullsize_cfg3.log
