# ncu --set full of the Kerr-Schild K3 (config 4, first stage-1 update), with source-level samples
CMD="python bench.py --config 4 --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/ks_small.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_update" -c 2 -o gpurun_out/ks_k3 $CMD > gpurun_out/ks_k3_ncu.log 2>&1
echo "rc=$?"
if [ -f gpurun_out/ks_k3.ncu-rep ]; then
  ncu -i gpurun_out/ks_k3.ncu-rep --page raw --csv > gpurun_out/ks_k3.raw.csv 2>/dev/null
  ncu -i gpurun_out/ks_k3.ncu-rep --page source --csv --print-source cuda,sass --launch-skip 1 --launch-count 1 > gpurun_out/ks_k3_src.csv 2>/dev/null
  rm -f gpurun_out/ks_k3.ncu-rep
fi
