#!/bin/bash
# C1 launch list + --set full capture of every hot kernel (one launch each).
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
K='regex:seed_kernel|solo_kernel|resolve_kernel|align_kernel|prune_kernel'
B="python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 12 --csv \
    --log-file $O/launches_${TAG}_C1.csv $B > $O/ncu_l1_$TAG.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$K" -c 6 \
    -o $O/prof_${TAG}_C1 -f $B > $O/ncu_f1_$TAG.log 2>&1
