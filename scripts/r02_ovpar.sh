#!/bin/bash
# per-chunk global-table passes on the chunks' own streams (per-stage tables) vs one shared stream
O=gpurun_out; mkdir -p $O; : > $O/ovpar.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par11.log 2>&1; echo rc=$? >> $O/t_par11.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c2_full or c1" > $O/t_full11.log 2>&1; echo rc=$? >> $O/t_full11.log
for v in libsnapb200.so variants/libsnapb200_ovstream.so; do
  lib=$PWD/paper_1111_5572_b200/lib/$v
  SNAP_B200_LIB=$lib timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 6 2>&1 | grep chunk | sed "s|^|$(basename $lib) |" >> $O/ovpar.log
  SNAP_B200_LIB=$lib timeout 600 python scripts/e2e_probe.py --config C1 --reads 1000000 --calls 8 2>&1 | grep chunk | sed "s|^|$(basename $lib) C1 |" >> $O/ovpar.log
done
SA_DEBUG_TIMELINE=1 timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 1 > $O/timeline_ovpar.log 2>&1
