#!/bin/bash
# GPU suite + C2 bench line (run under gpurun)
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/gputest_$TAG.log
timeout 900 python bench.py --steps 10 > $O/bench_$TAG.json 2> $O/bench_$TAG.err
