# the whole GPU suite + smoke + two default bench lines
set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=12 > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$?
tail -22 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
for r in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_r$r.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench_r$r.json').read().strip().splitlines()[-1]);print($r, round(d['ms_per_step'],2), d['clocks'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])"
done
