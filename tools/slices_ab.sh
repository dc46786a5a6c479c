#!/bin/bash
# Slices per query group for 10k-query batches over ~1M-row databases (configs 2 and 3): XFBQ_UMMA_SLICES forced vs the planner.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/slices_ab_r2e.log
: > $O
for shape in "1000000 128 100" "1200000 200 10" "1000000 256 100"; do
  for S in 0 2 3 7 11 15; do
    echo "== n dim k = $shape  slices=$S" >> $O
    if [ $S = 0 ]; then timeout 600 python tools/batch_sweep.py $shape 2500,5000,10000 >> $O 2>&1
    else XFBQ_UMMA_SLICES=$S timeout 600 python tools/batch_sweep.py $shape 2500,5000,10000 >> $O 2>&1; fi
  done
done
python - <<'PY'
import json
cur=None; tab={}
for l in open('gpurun_out/slices_ab_r2e.log'):
    if l.startswith('=='):
        p=l.split(); cur=(p[5],p[6],p[7],p[8]); continue
    try: d=json.loads(l)
    except Exception: continue
    tab.setdefault((cur[0],cur[1],cur[2],d['nq']),{})[cur[3]]=(d['call_ms'],d['parts'])
for k,v in tab.items(): print(k, v)
PY
