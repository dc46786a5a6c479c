run() { python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras "$@" 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), d['ms_per_step'], d['batch_scan']['kernel_ms'], d['config']['plan']['engine'])"; }
for nq in 17 32 48 64 96; do
  for e in umma imma; do echo -n "nq=$nq $e: "; XFBQ_ENGINE=$e run --nq $nq; done
done
