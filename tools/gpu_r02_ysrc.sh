# source-level stall samples of the first y sweep at 512^3 (cuda,sass export), the report deleted on the box
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain_y.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march --launch-skip 1 -c 1 -o /tmp/prof_y -f $CMD > gpurun_out/ncu_y.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_y.ncu-rep --page source --csv --print-source cuda,sass > /tmp/y_src.csv 2>/dev/null
python tools/line_stalls.py /tmp/y_src.csv 60 > gpurun_out/y_line_stalls.txt
python tools/sass_mix.py <(ncu -i /tmp/prof_y.ncu-rep --page source --csv --print-source sass) 134217728 > gpurun_out/y_sass_mix.txt 2>&1
gzip -c /tmp/y_src.csv > gpurun_out/y_src.csv.gz; ls -la gpurun_out/y_src.csv.gz
