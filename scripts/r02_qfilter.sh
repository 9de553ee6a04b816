#!/bin/bash
# q-gram filter: parity (every C3 and C4 read, parity suites) and C3/C4 timing vs the filter off
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu -k "c3 or c4" > $O/t_c34.log 2>&1; echo rc=$? >> $O/t_c34.log
bash scripts/variants.sh --steps 3 --config C3 > $O/variants_c3.log 2>&1
bash scripts/variants.sh --steps 3 --config C4 > $O/variants_c4.log 2>&1
