#!/bin/bash
# GPU suite + C2/C1 bench lines after a kernel change (run under gpurun).
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/gputest_$TAG.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 900 python bench.py --config C1 --steps 10 --no-cpu-baseline > $O/bench_${TAG}_C1.json 2> $O/bench_${TAG}_C1.err
