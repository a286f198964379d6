# 9-10 fewer FP64 instructions per cell and sweep (WENO5 C1/E1 factor on p02, HLL c = a sL, flat
# fast-speed Q in one FMA): GPU parity file, then a bench A/B against the previous code (fpold)
set -x
# (parity: the first run of this script, 49 passed incl. full size)

for r in 1 2 3; do
  for v in "" fpold; do
    ECHO_LIB_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/fp_${v:-default}_$r.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/fp_${v:-default}_$r.json').read().strip().splitlines()[-1]);print('${v:-default}', $r, round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
