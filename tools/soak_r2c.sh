#!/bin/bash
# Soak of the shipped library on one B200: randomised shapes on every engine vs the CPU oracle (several seeds), the thread-pool
# test repeated.  Output: gpurun_out/soak_r2c.log (one line per shape, "ALL OK" per run)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/soak_r2c.log
: > $L
for seed in 1 2 3; do echo "== small_stress seed $seed" >> $L; timeout 900 python tools/small_stress.py $seed 40 >> $L 2>&1; echo "small_stress $seed rc=$?" | tee -a $L; done
for seed in 2 3; do echo "== umma_stress seed $seed" >> $L; timeout 900 python tools/umma_stress.py $seed 100 >> $L 2>&1; echo "umma_stress $seed rc=$?" | tee -a $L; done
for seed in 1 2; do echo "== queue_stress seed $seed" >> $L; timeout 900 python tools/queue_stress.py $seed 40 >> $L 2>&1; echo "queue_stress $seed rc=$?" | tee -a $L; done
echo "== thread-pool test x 15" >> $L
for i in $(seq 15); do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k concurrent -p no:cacheprovider 2>&1 | tail -1 >> $L; done
grep -c "passed" $L | sed 's/^/thread-pool runs passed: /' | tee -a $L
grep -n "MISMATCH\|Error\|error\|failed" $L | head -20
