#!/bin/bash
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plainz.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sweep" -c 3 -o gpurun_out/profz $CMD > gpurun_out/ncuz.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncuz.log
