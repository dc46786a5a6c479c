#!/bin/bash
# A/B of the slice planner's first-wave fill (XFBQ_UMMA_FILL=0: slices of at least 512 tiles as before) on mid-size databases.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/fill_ab_r2c.log
: > $O
for shape in "2500000 256" "5000000 256" "4000000 1024" "3000000 512"; do
  for fill in 0 1; do
    echo "== n dim = $shape  XFBQ_UMMA_FILL=$fill" >> $O
    XFBQ_UMMA_FILL=$fill timeout 600 python tools/batch_sweep.py $shape 100 1,32,64,128,256,512,1024 >> $O 2>&1
  done
done
cut -c1-200 $O
