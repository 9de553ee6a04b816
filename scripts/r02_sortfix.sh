#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > $O/t_par13.log 2>&1; echo rc=$? >> $O/t_par13.log
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c2_full or c3" > $O/t_full13.log 2>&1; echo rc=$? >> $O/t_full13.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > $O/b_c2s.json 2>/dev/null
