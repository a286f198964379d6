# the whole GPU suite (as the driver runs it), then a default bench line
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/suite.log 2>&1
echo "suite rc=$?"
tail -25 gpurun_out/suite.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_suite.json 2> gpurun_out/bench_suite.err
echo "bench rc=$?"; tail -1 gpurun_out/bench_suite.json | head -c 600
