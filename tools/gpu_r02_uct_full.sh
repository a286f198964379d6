# UCT full-size 10-step parity (configs 1, 4), then ncu --set full of the UCT kernels at 512^3
set -x
export ECHO_PARITY_LOG=$PWD/gpurun_out/parity_uct_full.jsonl; rm -f $ECHO_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -s -k uct > gpurun_out/pytest_uct_full.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/pytest_uct_full.log
CMD="python bench.py --divb 2 --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/uct_plain.json 2>&1 && \
ncu --set full --clock-control none -k regex:"k_uct_emf|k_uct_cell|k_uct_induct|k_march" -c 7 \
  -o gpurun_out/prof_uct $CMD > gpurun_out/ncu_uct.log 2>&1
echo "ncu rc=$?"
if [ -f gpurun_out/prof_uct.ncu-rep ]; then
  ncu -i gpurun_out/prof_uct.ncu-rep --page raw --csv > gpurun_out/prof_uct.raw.csv 2>/dev/null
  rm -f gpurun_out/prof_uct.ncu-rep
fi
