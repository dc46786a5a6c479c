#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 1 2 3 4; do timeout 300 python bench.py --no-cpu-baseline --no-extras 2>gpurun_out/bench$i.err | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['batch_scan']['kernel_ms'], d['e2e']['value'], d['clocks'])"; done
tail -3 gpurun_out/bench1.err
