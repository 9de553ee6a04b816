#!/bin/bash
# global-table kernel pick_best with 4 candidates per lane in flight
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -q -x -m gpu > $O/t_par12.log 2>&1; echo rc=$? >> $O/t_par12.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c2_full or c3" > $O/t_full12.log 2>&1; echo rc=$? >> $O/t_full12.log
bash scripts/variants.sh --steps 10 > $O/variants_c2.log 2>&1
bash scripts/variants.sh --steps 3 --config C3 > $O/variants_c3.log 2>&1
