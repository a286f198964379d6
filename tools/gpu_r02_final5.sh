# End of round 2, library rebuilt from source: the ncu launch list of the default bench command
# (taken after the same command exited 0 without ncu), the UCT / rec-6 / config-4 bench lines,
# and the one-GPU z-slab decomposition line (f1's own cost on one device)
set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_final5_short.json 2> gpurun_out/bench_final5_short.err; echo bench_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final5.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_final5.log 2>&1; echo ncu_rc=$?
for a in "--divb 2" "--rec 6" "--config 4" "--decomp --slabs 2"; do
  n=$(echo $a | tr -d ' -')
  timeout 600 python bench.py $a --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_final5_$n.json 2>/dev/null; echo "$a rc=$?"
done
for f in gpurun_out/bench_final5*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step'],2), '%.3e'%d['value'], d['clocks']['sm_mhz'])"; done
