# rec = 6 (characteristic-wise WENO5, A44): GPU parity, then the bench lines (default and --rec 6)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug.py -x -q > gpurun_out/pytest_rec6.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_rec6.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --rec 6 > gpurun_out/bench_rec6.json 2> gpurun_out/bench_rec6.err; echo rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$?
tail -1 gpurun_out/bench_rec6.json; tail -1 gpurun_out/bench_default.json
