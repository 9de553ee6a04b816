# bench sweep over library variants: run_variants.sh TAG CONFIGS VARIANT...
TAG=$1; shift; CFGS=$1; shift
O=gpurun_out
for cfg in $CFGS; do
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L="SNAP_B200_LIB=paper_1111_5572_b200/lib/variants/libsnapb200_$v.so"; fi
  echo "== $cfg $v" >> $O/bench_$TAG.txt
  env $L timeout 600 python bench.py --config $cfg --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['overflow_kernel_ms'],3))" >> $O/bench_$TAG.txt 2>&1
done; done
