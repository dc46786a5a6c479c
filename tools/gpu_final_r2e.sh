#!/bin/bash
# Final evidence of round 2 on the shipped library: both bench arms, launch list of the bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r2e.json 2> gpurun_out/bench_ref_r2e.err; echo "ref rc=$?"
timeout 600 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo "bench rc=$?"
cut -c1-300 gpurun_out/bench_r2e.json
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum -c 800 --csv --log-file gpurun_out/launches_r2e_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2e.log 2>&1; echo "launch list rc=$?"
python tools/batch_sweep.py 10000000 256 100 > gpurun_out/sweep_10m_256_r2e.jsonl 2>&1
python tools/batch_sweep.py 1000000 256 100 > gpurun_out/sweep_1m_256_r2e.jsonl 2>&1
python tools/batch_sweep.py 1000000 768 100 1,16,64,1024,10000 > gpurun_out/sweep_1m_768_r2e.jsonl 2>&1
