run() { python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['batch_scan']['kernel_ms'], d['config']['plan']['engine'])"; }
timeout 100 python tools/umma_check.py | tail -1
echo -n "cfg1: "; run --n 100000 --dim 128 --doc-bits 4 --nq 100 --k 10
echo -n "cfg2: "; run --n 1000000 --dim 128 --doc-bits 3
echo -n "n=1.25M: "; run --n 1250000
echo -n "cfg4: "; run
echo -n "1M nq1000: "; run --n 1000000 --dim 128 --doc-bits 3 --nq 1000
