# y/z 8 lines x 8 cells (2 warps, CTA barriers) at 6 and 7 CTAs/SM against the default 8 x 4 (1 warp)
set -x
timeout 300 python -m pytest tests/test_gpu_slab.py -q -k destroy > gpurun_out/pytest_destroy.log 2>&1; echo destroy_rc=$?; tail -2 gpurun_out/pytest_destroy.log
for v in yz886 yz887; do
  ECHO_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_and_stage or degenerate" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"
done
for r in 1 2; do
  for v in "" yz886 yz887; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/h_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/h_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
