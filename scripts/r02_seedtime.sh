#!/bin/bash
# Seed / solo / resolve kernel time and DRAM bytes per library variant (C2, one device launch each).
O=gpurun_out; mkdir -p $O
for so in paper_1111_5572_b200/lib/libsnapb200.so paper_1111_5572_b200/lib/variants/*.so; do
  echo "== $so"
  SNAP_B200_LIB=$PWD/$so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,dram__bytes_read.sum,smsp__inst_executed.sum \
    --clock-control none -k 'regex:seed_kernel|solo_kernel|resolve_kernel' -c 3 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' '{print $5, $13, $15}'
done > $O/seedtime.log 2>&1
