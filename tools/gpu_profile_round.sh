#!/bin/bash
# Round evidence (1 GPU): plain bench, ncu launch list of the bench command, one
# ncu --set full capture of the sweeps + update at 512^3.  Summaries go to
# profiles/ via tools/summarize_profiles.py (run on the CPU side).
mkdir -p gpurun_out
python -m paper_1810_04597_b200.build > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
$CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -c 4 \
  -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
