#!/bin/bash
O=gpurun_out; mkdir -p $O
bash scripts/variants.sh --steps 3 --config C4 > $O/variants_c4.log 2>&1
