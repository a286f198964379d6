# characteristic-wise WENO5 (rec 6) sweeps: CTAs/SM of the y/z sweeps (6 default: 240 registers;
# 10; 12: 160 registers, spill-free) and of the x sweep (3 default: 164; 4: 128), parity + A/B
set -x
for v in r6both; do
  ECHO_LIB_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rec6 or mp5 or switch or full_size_sampled" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest_rc=$?"
  tail -1 gpurun_out/pytest_$v.log
done
for r in 1 2; do
  for v in "" r6yz10 r6yz12 r6x4 r6both; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --rec 6 --steps 6 --warmup 3 --no-cpu > gpurun_out/r6_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/r6_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
