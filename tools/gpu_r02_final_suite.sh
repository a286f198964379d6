# the whole GPU suite + smoke + the driver-style bench line (K = 20, W = 5)
set -x
export ECHO_PARITY_LOG=$PWD/gpurun_out/parity_final.jsonl; rm -f $ECHO_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest_rc=$?
tail -18 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?
tail -1 gpurun_out/bench_final.json
