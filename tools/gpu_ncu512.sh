#!/bin/bash
# ncu of the three sweeps + update at 512^3 (config 3, the bench workload)
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain512.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -c 4 -o gpurun_out/prof512 $CMD > gpurun_out/ncu512.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu512.log
