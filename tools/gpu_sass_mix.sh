#!/bin/bash
# Dynamic SASS mix of the first stage's x and y sweeps at 512^3: ncu source page (SASS)
# exported on the GPU box as CSV (the report itself is too large to copy back).
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:"k_march" -c 2 -o gpurun_out/prof_mix -f $CMD \
  > gpurun_out/ncu_mix.log 2>&1
for i in 0 1; do
  ncu -i gpurun_out/prof_mix.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 \
    > gpurun_out/sass_mix_$i.csv 2>/dev/null
done
rm -f gpurun_out/prof_mix.ncu-rep
ls -la gpurun_out
