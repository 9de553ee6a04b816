#!/bin/bash
# Compare experimental library builds (lib/variants/) on the C1 bench.
cd "$(dirname "$0")/.."
for so in paper_1111_5572_b200/lib/libsnapb200.so paper_1111_5572_b200/lib/variants/*.so; do
  SNAP_B200_LIB=$PWD/$so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | \
    python -c "import json,sys,os; d=json.loads(sys.stdin.read()); print(os.path.basename('$so'), round(d['value']/1e6,1), 'Mreads/s  kernel_ms', round(d['roofline']['kernel_ms'],3), ' e2e', round(d['e2e']['value']/1e6,1))"
done
