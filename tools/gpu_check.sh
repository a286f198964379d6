#!/bin/bash
# First-contact GPU check: environment, smoke, GPU tests, short bench.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --n 256 256 256 > gpurun_out/bench256.log 2>&1; echo "rc=$?" >> gpurun_out/bench256.log
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-steps 1 > gpurun_out/bench512.log 2>&1; echo "rc=$?" >> gpurun_out/bench512.log
