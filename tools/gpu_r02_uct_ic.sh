# UCT induction / cell-update marches: planes per thread (ECHO_ZSEG_IC 16 default, 8, 4) and the
# induction compiled for 8 CTAs/SM (ib8, then the default); round 2: ib6, ib12, cell at 8 CTAs/SM (cb8); UCT parity of the variants, then an alternated bench A/B
set -x
for v in ib12 cb8; do
  ECHO_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_uct.py -q -x > gpurun_out/pytest_uct_$v.log 2>&1; echo "$v pytest_rc=$?"
  tail -1 gpurun_out/pytest_uct_$v.log
done
for r in 1 2; do
  for v in "" ib6 ib12 cb8; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --divb 2 --steps 6 --warmup 3 --no-cpu > gpurun_out/ic_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ic_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
