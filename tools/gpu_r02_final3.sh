# Final code of the session (after the UCT induction and rec-6 occupancy changes): the whole GPU
# suite, smoke, the driver-style bench line, and the UCT / rec-6 / config-4 bench lines
set -x
export ECHO_PARITY_LOG=$PWD/gpurun_out/parity_final3.jsonl; rm -f $ECHO_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final3.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_final3.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo bench_rc=$?
for a in "--divb 2" "--rec 6" "--config 4"; do
  n=$(echo $a | tr -d ' -')
  timeout 600 python bench.py $a --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_final3_$n.json 2>/dev/null; echo "$a rc=$?"
done
for f in gpurun_out/bench_final3*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step'],2), '%.3e'%d['value'], d['clocks']['sm_mhz'])"; done
