#!/bin/bash
# L2 fetch-granularity hint (SA_L2_FETCH -> cudaLimitMaxL2FetchGranularity):
# C2 device/e2e rate and the seed kernel's DRAM bytes per setting.
TAG=${1:-r02x}
O=gpurun_out; mkdir -p $O
: > $O/l2fetch_$TAG.txt
for v in "" 32 64 128; do
  SA_L2_FETCH=$v timeout 600 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L2_FETCH=$v', round(d['value']/1e6,1), 'M dev', round(d['e2e']['value']/1e6,1), 'M e2e kernel_ms', round(d['roofline']['kernel_ms'],3))" >> $O/l2fetch_$TAG.txt
done
for v in "" 32; do
  SA_L2_FETCH=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --clock-control none -k 'regex:seed_kernel|solo_kernel|align_kernel|prune_kernel|resolve_kernel' -c 40 --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/l2fetch_ncu_${TAG}_$v.csv 2>&1
done
