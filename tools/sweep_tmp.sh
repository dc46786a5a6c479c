#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 150 python tools/umma_check.py > gpurun_out/check.log 2>&1; echo "check rc=$?"; tail -2 gpurun_out/check.log
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/umma_stress.py > gpurun_out/stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/stress.log
b() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['batch_scan']['kernel_ms'], d['e2e']['value'])"; }
b XFBQ_MERGE_BOUNDED=0
b XFBQ_MERGE_BOUNDED=1
timeout 900 bash tools/bench_configs.sh > gpurun_out/configs.jsonl; cat gpurun_out/configs.jsonl
