#!/bin/bash
# C3 after the q-gram filter: launch list + full captures of the main and the global-table kernel
O=gpurun_out; mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:seed_kernel|align_kernel' -c 9 --csv \
    --log-file $O/launches_r02n_C3.csv $B > $O/ncu_l3n.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' -c 1 \
    -o $O/prof_r02n_C3main -f $B > $O/ncu_f3m.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' --launch-skip 1 -c 1 \
    -o $O/prof_r02n_C3slow -f $B > $O/ncu_f3s.log 2>&1
