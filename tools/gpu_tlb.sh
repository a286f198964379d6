#!/bin/bash
for n in "512 512 512" "512 256 1024" "512 128 2048" "512 64 4096"; do
  python bench.py --steps 2 --warmup 1 --no-cpu --n $n 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline']; s=r['kernel_share_of_step']; t=d['ms_per_step']
print('$n', 'ms/step %.1f'%t, {k: round(v*t/3,2) for k,v in s.items()})"
done
