# guard-band OOB-write checks on every path, UCT parity, then bench lines: UCT (--divb 2) and configs 1, 2, 4
set -x
timeout 900 python -m pytest tests/test_gpu_guards.py tests/test_gpu_uct.py tests/test_gpu_fused.py -x -q > gpurun_out/pytest_guards.log 2>&1; echo pytest_rc=$?
tail -6 gpurun_out/pytest_guards.log
for a in "--divb 2" "--config 1" "--config 2" "--config 4" "--config 0"; do
  n=$(echo $a | tr -d ' -')
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu $a > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo "$a rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_$n.json').read().strip().splitlines()[-1]);print('$a', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
done
