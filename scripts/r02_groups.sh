#!/bin/bash
# grouped pipeline (SA_PIPE_GROUP chunks per group for the listed reads' kernels)
O=gpurun_out; mkdir -p $O; : > $O/groups.log
for g in 1 2 4 8; do
  SA_PIPE_GROUP=$g timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep -i "chunk\|error\|Trace" | sed "s/^/G=$g /" >> $O/groups.log
done
for g in 4; do
  SA_PIPE_GROUP=$g timeout 900 python bench.py --steps 5 --no-cpu-baseline > $O/b_grp$g.json 2> $O/b_grp$g.err; echo "bench G=$g rc=$?" >> $O/groups.log
  SA_PIPE_GROUP=$g timeout 600 python scripts/e2e_probe.py --config C1 --reads 1000000 --calls 8 2>&1 | grep chunk | sed "s/^/C1 G=$g /" >> $O/groups.log
done
SA_PIPE_GROUP=4 SA_DEBUG_TIMELINE=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_grp4.log 2>&1
