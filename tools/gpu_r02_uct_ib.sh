# the induction march: compiled for 8 CTAs/SM (default, 64 registers) against ptxas's own budget
# (ib0, 86 registers); alternated UCT bench at 512^3
set -x
for r in 1 2 3; do
  for v in "" ib0; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --divb 2 --steps 6 --warmup 3 --no-cpu > gpurun_out/ib_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ib_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
