#!/bin/bash
O=gpurun_out; mkdir -p $O; : > $O/ovrule.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c3 or c2_full" > $O/t_ov.log 2>&1; echo rc=$? >> $O/t_ov.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/t_par6.log 2>&1; echo rc=$? >> $O/t_par6.log
timeout 600 python scripts/e2e_probe.py --config C3 --reads 500000 --calls 4 2>&1 | grep chunk >> $O/ovrule.log
timeout 600 python scripts/e2e_probe.py --config C2 --reads 10000000 --calls 4 2>&1 | grep chunk >> $O/ovrule.log
