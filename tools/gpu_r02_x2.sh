# the x sweep with two cells per lane (march_pair.cuh): bitwise against the one-cell x sweep
# (variant xold), the GPU parity file, then a bench A/B (default / xold / CTAs per SM 3 and 5)
set -x
for v in "" xold; do
  ECHO_LIB_VARIANT=$v timeout 600 python tools/variant_bitwise.py > gpurun_out/bw_${v:-default}.txt 2>&1; echo "bw $v rc=$?"
done
diff gpurun_out/bw_default.txt gpurun_out/bw_xold.txt && echo BITWISE_SAME
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity_x2.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_parity_x2.log
for r in 1 2; do
  for v in "" xold x2b3 x2b5; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/x2_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/x2_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
