#!/bin/bash
# C2 e2e: pipeline stages x chunk size
O=gpurun_out; mkdir -p $O; : > $O/stages2.log
for v in libsnapb200.so variants/libsnapb200_st10.so variants/libsnapb200_st16.so; do for c in 425984 655360 1048576 1572864; do
  lib=$PWD/paper_1111_5572_b200/lib/$v
  SNAP_B200_LIB=$lib SA_CHUNK_READS=$c timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 5 2>&1 | grep chunk | sed "s|^|$(basename $lib) |" >> $O/stages2.log
done; done
