# occupancy knobs of the KS and UCT kernels (prebuilt variants): config-4 and UCT bench A/B
mkdir -p gpurun_out/knobs
for r in 1 2; do
  for v in "" ksu3 ksx5 ksx3; do
    ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu > gpurun_out/knobs/c4_${v:-default}_$r.json 2>/dev/null
    tail -1 gpurun_out/knobs/c4_${v:-default}_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c4 ${v:-default}', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
  for v in "" emf2 emf4; do
    ECHO_LIB_VARIANT="$v" timeout 600 python bench.py --divb 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/knobs/uct_${v:-default}_$r.json 2>/dev/null
    tail -1 gpurun_out/knobs/uct_${v:-default}_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('uct ${v:-default}', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['roofline']['kernel_share_of_step'])"
  done
done
