# parity subset + C2 variants: mask LV on/off, pruning batch modes
TAG=${1:-e}
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -x -q -m gpu > $O/gputest_$TAG.log 2>&1
echo "rc=$?" >> $O/gputest_$TAG.log
SA_PB_MODE=2 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "c2_full or c1_full" > $O/gputest_full_$TAG.log 2>&1
echo "rc=$?" >> $O/gputest_full_$TAG.log
for v in "SA_PB_MODE=2" "SA_PB_MODE=1" "SA_PB_MODE=2 SNAP_B200_LIB=paper_1111_5572_b200/lib/variants/libsnapb200_nomask.so"; do
  echo "== $v" >> $O/bench_$TAG.txt
  env $v timeout 600 python bench.py --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['overflow_kernel_ms'],3))" >> $O/bench_$TAG.txt 2>&1
done
env SA_PB_MODE=2 timeout 600 python bench.py --config C1 --steps 10 --no-cpu-baseline 2>&1 | tail -1 >> $O/bench_$TAG.txt
