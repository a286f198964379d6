#!/bin/bash
# Build tuning variants of the library (sweep line geometry), CPU side:
#   tools/build_variants.sh name "-DECHO_X_GEOM=4,64,3 -DECHO_YZ_GEOM=8,32,2" [name "defs"] ...
set -e
while [ $# -ge 2 ]; do
  python -m paper_1810_04597_b200.build --variant "$1" $2 > /dev/null &
  shift 2
done
wait
ls -la paper_1810_04597_b200/*.so
