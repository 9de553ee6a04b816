#!/bin/bash
# C2 e2e vs pipeline stages (copy buffers in flight), with the timeline of the last call
O=gpurun_out; mkdir -p $O; : > $O/stages.log
for v in "" variants/libsnapb200_st10.so variants/libsnapb200_st16.so; do
  lib=$PWD/paper_1111_5572_b200/lib/${v:-libsnapb200.so}
  SNAP_B200_LIB=$lib timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep chunk | sed "s|^|$(basename $lib) |" >> $O/stages.log
  SNAP_B200_LIB=$lib SA_DEBUG_TIMELINE=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_$(basename $lib .so).log 2>&1
done
