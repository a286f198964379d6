# Kerr-Schild K3 with the metric records staged in shared memory: KS parity tests, then config-4 bench A/B
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_fullsize.py -x -q -k "4 or torus or ks or KS" 2>&1 | tail -4
mkdir -p gpurun_out/ks_k3_ab
for r in 1 2; do
  for v in kssm0 "" kssm3; do
    ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/ks_k3_ab/${v:-new}_$r.json 2>/dev/null
    tail -1 gpurun_out/ks_k3_ab/${v:-new}_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('${v:-new}', d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
