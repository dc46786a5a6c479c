#!/bin/bash
cd "$(dirname "$0")/.."
b() { echo -n "$* : "; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['batch_scan']['kernel_ms'])"; }
b A=1
b XFBQ_UMMA_SLICES=7
b XFBQ_UMMA_SLICES=15
b XFBQ_UMMA_SLICES=22
b XFBQ_UMMA_CAP=512
b XFBQ_UMMA_CAP=160
b XFBQ_UMMA_HIST_SHIFT=1
b XFBQ_UMMA_HIST_SHIFT=3
b XFBQ_SEED_BELOW4=6
b XFBQ_SEED_BELOW4=12
b A=1
