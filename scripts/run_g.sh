# parity subset + eager-probe sweep on C2 and C1
TAG=${1:-g}
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solo.py -x -q -m gpu > $O/gputest_$TAG.log 2>&1
echo "rc=$?" >> $O/gputest_$TAG.log
for cfg in C2 C1; do
for v in 0 3 4 5 6; do
  echo "== $cfg eager=$v" >> $O/bench_$TAG.txt
  SA_EAGER_PROBES=$v timeout 600 python bench.py --config $cfg --steps 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['overflow_kernel_ms'],3))" >> $O/bench_$TAG.txt 2>&1
done; done
