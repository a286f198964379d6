#!/bin/bash
# GPU side: short 512^3 bench of each prebuilt variant (libecho_b200_<name>.so) + the default lib.
mkdir -p gpurun_out
for v in "" "$@"; do
  ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/var_${v:-default}.json 2> gpurun_out/var_${v:-default}.err
  echo "variant=${v:-default} rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/var_${v:-default}.json')); print(d['ms_per_step'], d['roofline']['kernel_share_of_step'], d['roofline']['avg_launch_ms'])" 2>/dev/null
done
