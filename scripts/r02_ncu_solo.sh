#!/bin/bash
# --set full capture of one kernel (default solo_kernel) at C2, one launch.
TAG=${1:-r02}; K=${2:-solo_kernel}
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$K" -c 1 \
    -o $O/prof_${TAG}_${K} -f $B > $O/ncu_${TAG}_${K}.log 2>&1
