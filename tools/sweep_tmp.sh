timeout 300 python tools/umma_check.py 2>&1 | tail -1
for cfg in "XFBQ_SEED_SPLIT=1" "XFBQ_SEED_SPLIT=2" "XFBQ_SEED_SPLIT=4" "XFBQ_SEED_SPLIT=1 XFBQ_SAMPLE=262144" "XFBQ_SEED_SPLIT=2 XFBQ_SAMPLE=65536" "XFBQ_SEED_SPLIT=1 XFBQ_SAMPLE=32768"; do
  echo "== $cfg"; env $cfg timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['batch_scan'])"
done
