#!/bin/bash
# ncu --set full of the first stage's three sweeps + update at 512^3 (bench workload), source-level
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -c 4 -o gpurun_out/prof_sweeps -f $CMD > gpurun_out/ncu_sweeps.log 2>&1
echo "ncu rc=$?"
