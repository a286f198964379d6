# WENO5 normalisation by two independent reciprocals (-DECHO_WENO_TWO_RCP, variant rcp2) against one
# shared reciprocal (default): parity of the variant, then an alternated bench A/B
set -x
ECHO_LIB_VARIANT=rcp2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_rcp2.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_rcp2.log
for r in 1 2 3; do
  for v in "" rcp2; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/rc_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/rc_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
