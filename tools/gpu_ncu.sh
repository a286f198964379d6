#!/bin/bash
# ncu capture of the sweep + update kernels on a 256^3 config-3 grid (1 GPU).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --n 256 256 256"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -c 4 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu.log
