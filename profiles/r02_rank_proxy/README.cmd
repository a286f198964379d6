# Per-rank proxy of the z-slab strong scaling on one GPU: ONE slab of an N-way decomposition of
# 512^3 (512 x 512 x 512/N planes) and of the paper's 1024^3 on 8 GPUs (1024 x 1024 x 128), run
# as a periodic slab that is its own neighbour (its 6 ghost planes per side filled by a local
# copy exchange before every stage, the ghost-plane sweeps included): the compute side of one
# rank's step; the NVLink transfer itself is not in it (scaling_model.py: hidden by the overlap)
set -x
for n3 in 512 256 128 64; do
  timeout 600 python bench.py --decomp --slabs 1 --n 512 512 $n3 --steps 8 --warmup 3 --no-cpu > gpurun_out/rank_512_$n3.json 2>gpurun_out/rank_512_$n3.err
  tail -1 gpurun_out/rank_512_$n3.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('512x512x$n3', d['ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --decomp --slabs 1 --n 1024 1024 128 --steps 5 --warmup 2 --no-cpu > gpurun_out/rank_1024_128.json 2>gpurun_out/rank_1024_128.err
tail -1 gpurun_out/rank_1024_128.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('1024x1024x128', d['ms_per_step'], d['clocks']['sm_mhz'])"
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > gpurun_out/rank_single.json 2>/dev/null
tail -1 gpurun_out/rank_single.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('single 512^3', d['ms_per_step'], d['clocks']['sm_mhz'])"
