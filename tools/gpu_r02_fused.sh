# fused update + x sweep (opt-in ECHO_FUSED_UPDATE=1): correctness, then A/B bench against the separate kernels
set -x
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_debug.py tests/test_gpu_advance.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_fused.log
for r in 1 2; do
  ECHO_FUSED_UPDATE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_fused_$r.json 2> gpurun_out/bench_fused_$r.err; echo rc=$?
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_unfused_$r.json 2> gpurun_out/bench_unfused_$r.err; echo rc=$?
done
for f in gpurun_out/bench_*fused_*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['ms_per_step'],d['roofline']['kernel_share_of_step'],d['clocks'])"; done
