# The transposed line-major y/z sweeps (ECHO_YZ_TRANS, variant libecho_b200_yzt.so): parity, then a bench A/B
set -x
ECHO_LIB_VARIANT=yzt timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -x -q 2>&1 | tail -4
mkdir -p gpurun_out/yzt_ab
for r in 1 2; do
  for v in "" yzt; do
    ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/yzt_ab/${v:-default}_$r.json 2>/dev/null
    tail -1 gpurun_out/yzt_ab/${v:-default}_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('${v:-default}', d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
