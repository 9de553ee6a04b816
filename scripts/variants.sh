#!/bin/bash
# Compare experimental library builds (lib/variants/) on the C1 bench.
# Extra env settings per run: VARIANT_ENVS="A=1 B=2" applies to every run.
cd "$(dirname "$0")/.."
shopt -s nullglob
for so in paper_1111_5572_b200/lib/libsnapb200.so paper_1111_5572_b200/lib/variants/*.so; do
  env $VARIANT_ENVS SNAP_B200_LIB=$PWD/$so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" 2>&1 | tail -1 | \
    python -c "import json,sys,os; d=json.loads(sys.stdin.read()); print(os.path.basename('$so'), '$VARIANT_ENVS', round(d['value']/1e6,3), 'Mreads/s  kernel_ms', round(d['roofline']['kernel_ms'],3), 'ovf_ms', round(d['roofline']['overflow_kernel_ms'],3), ' e2e', round(d['e2e']['value']/1e6,1), 'ev_ms', round(d['e2e']['event_ms_per_step'],3))"
done
