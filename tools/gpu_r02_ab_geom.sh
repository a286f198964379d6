# y/z geometry A/B on one box: default (8 lines x 4 cells, 12 CTA/SM), 8x4 at 14 CTA/SM,
# 4 x 8 at 12, 4 x 8 at 16 with tight rings; alternated twice; plus a quick parity check of each
set -x
for v in yzb14 yz4812 yz4816t; do
  ECHO_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "rhs_and_stage or degenerate or multistep_parity" > gpurun_out/pytest_$v.log 2>&1; echo "$v pytest rc=$?"
done
for r in 1 2; do
  for v in "" yzb14 yz4812 yz4816t; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/g_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/g_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
