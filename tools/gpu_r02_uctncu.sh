# per-kernel durations of the UCT EMF kernels, old vs shared, in one ncu invocation
ncu --target-processes all --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__inst_executed_pipe_fp64.sum --clock-control none -k regex:"k_uct_emf" --csv \
  bash -c 'ECHO_LIB_VARIANT=uctold python tools/uct_emf_one_step.py; python tools/uct_emf_one_step.py' > gpurun_out/uct_emf_ncu.csv 2> gpurun_out/uct_emf_ncu.err
echo rc=$?
