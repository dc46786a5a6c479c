#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 150 python tools/umma_check.py > gpurun_out/check.log 2>&1; echo "check rc=$?"; tail -1 gpurun_out/check.log
timeout 300 python tools/umma_stress.py > gpurun_out/stress.log 2>&1; echo "stress rc=$?"; tail -1 gpurun_out/stress.log
bash tools/gpu_round.sh smoke tests bench ncu
timeout 900 bash tools/bench_configs.sh > gpurun_out/configs.jsonl; cat gpurun_out/configs.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -f -o gpurun_out/prof_seed \
   python bench.py --steps 1 --warmup 1 --nq 10000 --no-cpu-baseline --no-extras > gpurun_out/ncuseed.log 2>&1; echo "ncu seed rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_queue_kernel -s 2 -c 1 -f -o gpurun_out/prof_queue \
   python bench.py --steps 1 --warmup 1 --nq 10000 --no-cpu-baseline --no-extras > gpurun_out/ncuqueue.log 2>&1; echo "ncu queue rc=$?"
timeout 300 python tools/umma_profile.py 10000 10000000 256 100
for nq in 1 8; do timeout 300 python tools/small_batch.py $nq 50 2>&1 | tail -1; done
