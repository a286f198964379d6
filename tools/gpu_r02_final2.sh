# Final evidence of the session's code: the whole GPU suite, smoke, the driver-style bench line
# (K = 20, W = 5), the ncu launch list of a short bench, and one ncu --set full capture of the first
# stage's three sweeps + update at 512^3 (summarised on the box; the report is not copied back)
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/gpu_final2.txt 2>&1
export ECHO_PARITY_LOG=$PWD/gpurun_out/parity_final2.jsonl; rm -f $ECHO_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_final2.log 2>&1; echo pytest_rc=$?
tail -8 gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_final2.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench_rc=$?
tail -1 gpurun_out/bench_final2.json | cut -c1-400
CMD="python bench.py --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/bench_small2.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final2.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none -k regex:"k_march|k_update" -c 4 -o /tmp/prof_final2 -f $CMD > gpurun_out/ncu_full2.log 2>&1
echo "full rc=$?"
python tools/ncu_summary.py /tmp/prof_final2.ncu-rep > gpurun_out/kernels_final2.txt 2>&1
head -60 gpurun_out/kernels_final2.txt
