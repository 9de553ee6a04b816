#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root):
#   r02_full.sh TAG -- GPU suite, smoke, bench C2 (default, with the CPU
#   baseline), the reference arm, C0/C1/C3/C4 lines, whole-box mode on one
#   device, C4 launch list + full capture of the long-read kernel.
TAG=${1:-r02}
O=gpurun_out; mkdir -p $O
nvidia-smi -L > $O/host_$TAG.txt; nproc >> $O/host_$TAG.txt; free -g >> $O/host_$TAG.txt
timeout 2400 python -m pytest tests -x -q -m gpu > $O/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/gputest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
for c in C0 C1 C3 C4; do
  timeout 900 python bench.py --config $c --steps 5 > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err
done
timeout 900 python bench.py --box --box-devices 0,0 --config C1 --steps 5 > $O/bench_${TAG}_box00.json 2> $O/bench_${TAG}_box00.err
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:align_kernel' -c 12 --csv \
    --log-file $O/launches_${TAG}_C4.csv $B --config C4 > $O/ncu_l4_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:align_kernel' -c 1 \
    -o $O/prof_${TAG}_C4 -f $B --config C4 > $O/ncu_f4_$TAG.log 2>&1
