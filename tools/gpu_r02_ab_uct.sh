# UCT register budgets: default (UCT x sweep at 5 CTAs/SM), uctold (6, round 1), emf2 (EMF z-march at 2 CTAs/SM)
set -x
timeout 600 python -m pytest tests/test_gpu_uct.py -q -x > gpurun_out/pytest_uct.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_uct.log
for r in 1 2; do
  for v in "" uctold emf2; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --divb 2 --steps 6 --warmup 3 --no-cpu > gpurun_out/u_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/u_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
