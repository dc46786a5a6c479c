#!/bin/bash
# Soak of the final library of round 2 (planner changes in): randomised shapes on the planner's own plans vs the CPU oracle.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=gpurun_out/soak_r2e.log
: > $L
for seed in 21 22; do echo "== small_stress seed $seed" >> $L; timeout 900 python tools/small_stress.py $seed 40 >> $L 2>&1; echo "small_stress $seed rc=$?" | tee -a $L; done
for seed in 23 24; do echo "== queue_stress (default plans) seed $seed" >> $L; QS_DEFAULT_PLANS=1 timeout 900 python tools/queue_stress.py $seed 50 >> $L 2>&1; echo "queue_stress default $seed rc=$?" | tee -a $L; done
echo "== queue_stress (forced slices / rings / samples) seed 25" >> $L; timeout 900 python tools/queue_stress.py 25 40 >> $L 2>&1; echo "queue_stress 25 rc=$?" | tee -a $L
echo "== umma_stress seed 26" >> $L; timeout 900 python tools/umma_stress.py 26 100 >> $L 2>&1; echo "umma_stress 26 rc=$?" | tee -a $L
for i in $(seq 8); do timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k concurrent -p no:cacheprovider 2>&1 | tail -1 >> $L; done
grep -c "passed" $L | sed 's/^/thread-pool runs passed: /' | tee -a $L
grep -n "MISMATCH\|Error\|failed" $L | head -20
