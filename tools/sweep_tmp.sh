run() { python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['batch_scan']['kernel_ms'])"; }
timeout 100 python tools/umma_check.py 2>&1 | tail -1
echo -n "cfg1 "; run --n 100000 --dim 128 --doc-bits 4 --nq 100 --k 10
echo -n "cfg2 "; run --n 1000000 --dim 128 --doc-bits 3 --nq 10000 --k 100
echo -n "cfg3 "; run --n 1200000 --dim 200 --doc-bits 4 --nq 10000 --k 10
echo -n "cfg4 "; run
echo -n "cfg5b "; run --n 12500000 --dim 512 --doc-bits 4 --nq 1024 --k 1000
echo -n "1M x 128 nq 1000 "; run --n 1000000 --dim 128 --doc-bits 3 --nq 1000 --k 100
echo -n "3M x 256 k100 nq 2000 "; run --n 3000000 --nq 2000
echo -n "10M x 256 k100 nq 500 "; run --nq 500
