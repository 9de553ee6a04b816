#!/bin/bash
# long reads (non-seeded path) from pageable buffers: staged through pinned buffers
O=gpurun_out; mkdir -p $O; : > $O/c4pageable.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c4" > $O/t_c4p.log 2>&1; echo rc=$? >> $O/t_c4p.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/t_par10.log 2>&1; echo rc=$? >> $O/t_par10.log
P="timeout 600 python scripts/e2e_probe.py --config C4 --reads 50000 --calls 4"
$P --pageable 2>&1 | grep chunk >> $O/c4pageable.log
SA_NO_STAGING=1 $P --pageable 2>&1 | grep chunk | sed 's/^/nostaging /' >> $O/c4pageable.log
$P 2>&1 | grep chunk | sed 's/^/pinned /' >> $O/c4pageable.log
