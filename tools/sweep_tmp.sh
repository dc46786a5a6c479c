run() { python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['batch_scan']['kernel_ms'], d['config']['plan']['engine'])"; }
for n in 1250000 2500000 5000000; do
for smp in 16384 8192 4096 2048; do echo -n "n=$n sample=$smp: "; XFBQ_SAMPLE=$smp run --n $n; done
done
