# Kerr-Schild config 4: A/B of the x-sweep and update occupancy (spill-free register budgets)
set -x
ECHO_LIB_VARIANT= timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or 4-n" > gpurun_out/pytest_ks.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_ks.log
for r in 1 2 3; do
  for v in "" ksold ks4; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu > gpurun_out/k_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/k_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
