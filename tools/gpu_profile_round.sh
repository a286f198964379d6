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
# UCT (divb = 2): the edge-EMF kernel, first launch at 512^3
ncu --set full --clock-control none --import-source on -k regex:"k_uct_emf|k_uct_cell" -c 2 \
  -o gpurun_out/prof_uct python bench.py --divb 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_uct.log 2>&1
echo "uct rc=$?" >> gpurun_out/ncu_uct.log
# gpurun copies back <= 64 MiB: keep the raw-page CSV exports, drop the reports
for r in prof_round prof_uct; do
  if [ -f gpurun_out/$r.ncu-rep ]; then
    ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
    rm -f gpurun_out/$r.ncu-rep
  fi
done
