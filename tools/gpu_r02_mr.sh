# y/z sweeps with a __maxnreg__ register cap (146 / 141 / 136 registers used, spill-free: 13 / 14 / 15
# one-warp CTAs per SM) against the default launch bound (160 registers, 12 CTAs/SM)
set -x
ECHO_LIB_VARIANT=mr136 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_mr136.log 2>&1; echo "mr136 pytest_rc=$?"
tail -1 gpurun_out/pytest_mr136.log
for r in 1 2 3; do
  for v in "" mr152 mr144 mr136; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/mr_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/mr_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
