for cfg in "XFBQ_SAMPLE=131072" "XFBQ_SAMPLE=32768" "XFBQ_SAMPLE=16384 XFBQ_SEED_SPLIT=1" "XFBQ_SAMPLE=16384 XFBQ_SEED_SPLIT=4" "XFBQ_SAMPLE=8192 XFBQ_SEED_SPLIT=4" "XFBQ_SAMPLE=65536 XFBQ_SEED_SPLIT=4"; do
  echo "== $cfg"; env $cfg timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['batch_scan'])"
done
