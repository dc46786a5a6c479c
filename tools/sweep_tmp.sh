#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/ordered_db.py
for i in 1 0 1 0 1 0; do XFBQ_SEED_SPREAD=$i timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print($i, d['value'], d['ms_per_step'], d['batch_scan']['kernel_ms'], d['e2e']['value'])"; done
