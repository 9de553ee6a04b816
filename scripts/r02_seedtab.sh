#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par9.log 2>&1; echo rc=$? >> $O/t_par9.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu > $O/t_full9.log 2>&1; echo rc=$? >> $O/t_full9.log
bash scripts/variants.sh --steps 10 > $O/variants_c2.log 2>&1
bash scripts/variants.sh --steps 20 --config C1 > $O/variants_c1.log 2>&1
