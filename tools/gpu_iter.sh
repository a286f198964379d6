#!/bin/bash
# build -> GPU parity tests -> bench (512^3) ; args: pytest -k expression (optional)
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
K="${1:-not full_size}"
timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-steps 1 > gpurun_out/bench512.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench512.log
tail -c 2500 gpurun_out/bench512.log
