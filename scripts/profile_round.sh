#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   bench (C1, with the CPU baseline), the reference arm, the ncu launch list,
#   one ncu --set full capture of the seed and align kernels, and a bench line
#   per config.  Summarise afterwards here with scripts/ncu_summary.py.
TAG=${1:-r01d}
O=gpurun_out
set -x
python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref_$TAG.json 2> $O/bench_ref_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:seed_kernel|solo_kernel|align_kernel' -c 3 \
    -o $O/prof_c1_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_f_$TAG.log 2>&1
for c in C0 C2 C3 C4; do
    timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_${TAG}_$c.json 2> $O/bench_${TAG}_$c.err
done
