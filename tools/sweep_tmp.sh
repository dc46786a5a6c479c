#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 150 python tools/umma_check.py > gpurun_out/check.log 2>&1; echo "check rc=$?"; tail -2 gpurun_out/check.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/umma_stress.py > gpurun_out/stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/stress.log
timeout 900 bash tools/bench_configs.sh > gpurun_out/configs.jsonl; cat gpurun_out/configs.jsonl
