#!/bin/bash
# A/B of the sample shrink on small databases (XFBQ_SAMPLE_SHRINK=0: samples of at least 16k documents, i.e. no seeded
# thresholds and no queue kernel below 131k rows).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/small_db_ab_r2d.log
: > $O
for shape in "40000 128 10" "100000 128 10" "100000 256 100" "60000 768 10"; do
  for shrink in 0 1; do
    echo "== n dim k = $shape  arm=shrink$shrink" >> $O
    XFBQ_SAMPLE_SHRINK=$shrink timeout 600 python tools/batch_sweep.py $shape 32,100,256,1024,4096 >> $O 2>&1
  done
done
python - <<'PY'
import json
cur=None; tab={}
for l in open('gpurun_out/small_db_ab_r2d.log'):
    if l.startswith('=='):
        p=l.split(); cur=(p[5],p[6],p[7],p[8]); continue
    try: d=json.loads(l)
    except Exception: continue
    tab.setdefault((cur[0],cur[1],cur[2],d['nq']),{})[cur[3]]=(d['call_ms'],d['parts'])
for k,v in tab.items(): print(k, v)
PY
