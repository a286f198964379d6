#!/bin/bash
# Round-2 evidence (1 GPU): plain bench (default, K=20 W=5 like the driver), the ncu launch list of
# a short bench, one ncu --set full capture of the first stage's sweeps + update at 512^3 with the
# source pages of the y sweep exported (cuda,sass) for the per-phase stall analysis.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -c 4 \
  -o gpurun_out/prof_round $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
if [ -f gpurun_out/prof_round.ncu-rep ]; then
  ncu -i gpurun_out/prof_round.ncu-rep --page raw --csv > gpurun_out/prof_round.raw.csv 2>/dev/null
  for i in 0 1; do
    ncu -i gpurun_out/prof_round.ncu-rep --page source --csv --print-source cuda,sass --launch-skip $i --launch-count 1 \
      > gpurun_out/src_sweep_$i.csv 2>/dev/null
  done
  rm -f gpurun_out/prof_round.ncu-rep
fi
ls -la gpurun_out | tail -20
