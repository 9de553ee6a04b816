#!/bin/bash
# C3/C4 long-read evidence + gather ceiling (run under gpurun)
TAG=${1:-r02d}
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
K='regex:seed_kernel|solo_kernel|resolve_kernel|align_kernel|prune_kernel'
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gather_ceiling scripts/gather_ceiling.cu && \
  timeout 300 ./scripts/gather_ceiling 40 > $O/gather_ceiling_$TAG.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 12 --csv \
    --log-file $O/launches_${TAG}_C3.csv $B --config C3 > $O/ncu_l3_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 12 --csv \
    --log-file $O/launches_${TAG}_C4.csv $B --config C4 > $O/ncu_l4_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' -c 1 \
    -o $O/prof_${TAG}_C4 -f $B --config C4 > $O/ncu_f4_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' -c 2 \
    -o $O/prof_${TAG}_C3 -f $B --config C3 > $O/ncu_f3_$TAG.log 2>&1
