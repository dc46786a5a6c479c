for cfg in "XFBQ_UMMA_CAP=144" "XFBQ_UMMA_CAP=168" "XFBQ_UMMA_CAP=200" "XFBQ_UMMA_CAP=168 XFBQ_SAMPLE=8192" "XFBQ_UMMA_CAP=168 XFBQ_SAMPLE=32768"; do
  echo "== $cfg"; env $cfg timeout 100 python tools/umma_check.py 2>&1 | tail -1; env $cfg timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-extras 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['batch_scan'])"
done
