# transposed y/z geometry variants: bench A/B (default, 8 lines at 2 CTAs/SM, 4 lines at 6 and 5 CTAs/SM)
mkdir -p gpurun_out/yzt_ab
for r in 1 2; do
  for v in "" yzt2 yzt4 yzt45; do
    ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/yzt_ab/${v:-default}_b$r.json 2>/dev/null
    tail -1 gpurun_out/yzt_ab/${v:-default}_b$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('${v:-default}', d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
