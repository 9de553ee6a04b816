#!/bin/bash
# Seed-kernel grid (SA_SEED_GRID blocks of 64 reads, grid-stride beyond) at C2 and C1.
O=gpurun_out; mkdir -p $O
for g in 0 2368 9472 37888; do
  if [ $g = 0 ]; then E=""; else E="SA_SEED_GRID=$g"; fi
  echo "== $E"
  VARIANT_ENVS="$E" bash scripts/variants.sh --steps 10
  VARIANT_ENVS="$E" bash scripts/variants.sh --steps 20 --config C1
done > $O/seedgrid.log 2>&1
