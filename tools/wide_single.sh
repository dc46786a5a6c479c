#!/bin/bash
# Single queries on shapes the mma.sync engine does not take (more than 512 dims): XOR/POPC kernels vs the tcgen05 engine.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/wide_single_r2c.log
: > $O
for shape in "1000000 768" "8000000 768" "4000000 1024"; do
  for min in 2 1; do
    echo "== n dim = $shape  XFBQ_UMMA_MIN_NQ=$min" >> $O
    XFBQ_UMMA_MIN_NQ=$min timeout 600 python tools/batch_sweep.py $shape 100 1,2,4 >> $O 2>&1
  done
done
cat $O | cut -c1-260
