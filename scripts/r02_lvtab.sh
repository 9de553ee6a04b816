#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "lv_" > $O/t_lv.log 2>&1; echo rc=$? >> $O/t_lv.log
timeout 900 python -m pytest tests/test_gpu_solo.py -q -x -m gpu -k "warp_bitparallel" > $O/t_lvw.log 2>&1; echo rc=$? >> $O/t_lvw.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c4" > $O/t_c4.log 2>&1; echo rc=$? >> $O/t_c4.log
bash scripts/variants.sh --steps 3 --config C4 > $O/variants_c4.log 2>&1
