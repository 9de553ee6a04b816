#!/bin/bash
# Eager probes per read (SA_EAGER_PROBES) against the phase-synchronous solo kernel, C2 and C1.
O=gpurun_out; mkdir -p $O
for e in 4 5 6 8; do
  echo "== SA_EAGER_PROBES=$e"
  VARIANT_ENVS="SA_EAGER_PROBES=$e" bash scripts/variants.sh --steps 10
  VARIANT_ENVS="SA_EAGER_PROBES=$e" bash scripts/variants.sh --steps 20 --config C1
done > $O/eager.log 2>&1
