#!/bin/bash
# Phase-synchronous solo kernel: variants at C2 and C1 (lib/variants/*.so beside
# the default), then the whole GPU suite on the default library.
TAG=${1:-r02z}
O=gpurun_out; mkdir -p $O
bash scripts/variants.sh --steps 10 > $O/variants_${TAG}_c2.log 2>&1
bash scripts/variants.sh --steps 20 --config C1 > $O/variants_${TAG}_c1.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/gputest_$TAG.log
