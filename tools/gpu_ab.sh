#!/bin/bash
# build -> GPU parity tests -> bench default vs env variants ("NAME=VAL ..." args)
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-not full_size}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in "" "$@"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$v] rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['ms_per_step'], d['roofline']['kernel_share_of_step'], d['roofline']['avg_launch_ms'], d['counters'], d['gpu_launches'])" 2>&1 | tail -2
done
