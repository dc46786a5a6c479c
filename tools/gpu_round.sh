#!/bin/bash
# One GPU session: smoke, microbench, parity tests, bench, ncu launch list + full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [stages...]   stages: smoke micro tests bench ncu ncufull
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
STAGES="${@:-smoke micro tests bench ncu ncufull}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for s in $STAGES; do
  case $s in
    smoke) timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    micro2) timeout 120 tools/bin/microbench2 > gpurun_out/microbench2.jsonl 2>&1; echo "micro2 rc=$?" ;;
    ncumma) timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -f -o gpurun_out/prof_mma \
           python bench.py --steps 1 --warmup 1 --nq ${NQB:-10000} --no-cpu-baseline --no-extras > gpurun_out/ncumma.log 2>&1; echo "ncumma rc=$?" ;;
    q1) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/q1_launches.csv \
           python tools/small_batch.py 1 4 > gpurun_out/q1.log 2>&1; echo "q1 rc=$?"; timeout 300 python tools/small_batch.py 1 50 ; timeout 300 python tools/small_batch.py 8 50 ;;
    ncuq1) timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 7 -c 1 -f -o gpurun_out/prof_q1 \
           python tools/small_batch.py ${NQ:-8} 2 > gpurun_out/ncuq1.log 2>&1; echo "ncuq1 rc=$?" ;;
    bw) timeout 600 python tools/bw_probe.py > gpurun_out/bw_probe.log 2>&1; echo "bw rc=$?"; cat gpurun_out/bw_probe.log ;;
    micro) timeout 120 tools/bin/microbench > gpurun_out/microbench.jsonl 2>&1; echo "micro rc=$?" ;;
    tests) timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/pytest_gpu.log ;;
    bench) timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
           python bench.py --steps 1 --warmup 1 --nq 10000 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?" ;;
    ncufull) timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_topk -c 3 -f -o gpurun_out/prof_scan \
           python bench.py --steps 1 --warmup 1 --nq 512 --no-cpu-baseline > gpurun_out/ncufull.log 2>&1; echo "ncufull rc=$?" ;;
  esac
done
