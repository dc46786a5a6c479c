#!/bin/bash
# QPS of the BASELINE.json config shapes on one GPU (config 5 at 1/8 of its rows = one GPU's shard of eight).
# Usage (under gpurun): bash tools/bench_configs.sh > gpurun_out/configs.jsonl
cd "$(dirname "$0")/.."
run() { python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(json.dumps({'workload': d['config']['workload'], 'qps': d['value'], 'e2e_qps': d['e2e']['value'], 'ms_per_step': d['ms_per_step'], 'engine': d['config']['plan']['engine'], 'kernel_ms': d['batch_scan']['kernel_ms']}))"; }
run --n 100000 --dim 128 --doc-bits 4 --nq 100 --k 10
run --n 1000000 --dim 128 --doc-bits 3 --nq 10000 --k 100
run --n 1200000 --dim 200 --doc-bits 4 --nq 10000 --k 10
run --n 10000000 --dim 256 --doc-bits 4 --nq 10000 --k 100
run --n 12500000 --dim 512 --doc-bits 4 --nq 1024 --k 1000
run --n 12500000 --dim 512 --doc-bits 4 --nq 1 --k 1000
