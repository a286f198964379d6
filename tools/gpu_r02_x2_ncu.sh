# ncu --set full of the first x sweep: the two-cells-per-lane kernel (default, 4 CTAs/SM; x2b3) and the one-cell one (xold)
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
for v in "" x2b3 xold; do
  ECHO_LIB_VARIANT=$v $CMD > gpurun_out/plain_$v.json 2>&1 || continue
  ECHO_LIB_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_march" -c 1 -o gpurun_out/prof_x2_${v:-default} -f $CMD > gpurun_out/ncu_x2_${v:-default}.log 2>&1
  echo "ncu $v rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_x2_${v:-default}.ncu-rep
done
