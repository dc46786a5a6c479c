#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/sweep_tmp.py
timeout 150 python tools/umma_check.py > gpurun_out/check.log 2>&1; echo "check rc=$?"; tail -1 gpurun_out/check.log
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['batch_scan']['kernel_ms'], d['e2e']['value'])"; done
timeout 900 bash tools/bench_configs.sh
