# guard-band + UCT + fused tests on the default build, then an A/B/C of the y/z sweep variants
# (default: branch-free edge loads; noedge: round 1's branched edge loads; accregs: + old
# accumulator values in registers), alternated 3 times on one box
set -x
timeout 900 python -m pytest tests/test_gpu_guards.py tests/test_gpu_uct.py tests/test_gpu_fused.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_ab.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_ab.log
for r in 1 2 3; do
  for v in "" noedge accregs; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
