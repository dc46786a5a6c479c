#!/bin/bash
# A/B of the smallest database the queue kernel is used for (XFBQ_UMMA_QUEUE_MIN_N, default 2 000 000) on 0.5M-1.5M-row corpora.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/queue_min_ab_r2d.log
: > $O
for shape in "1000000 128" "1000000 256" "1000000 768" "500000 256" "1500000 512"; do
  for minn in 2000000 300000; do
    echo "== n dim = $shape  XFBQ_UMMA_QUEUE_MIN_N=$minn" >> $O
    XFBQ_UMMA_QUEUE_MIN_N=$minn timeout 600 python tools/batch_sweep.py $shape 100 32,64,256,512,1024,2048 >> $O 2>&1
  done
done
python - <<'PY'
import json
cur=None; tab={}
for l in open('gpurun_out/queue_min_ab_r2d.log'):
    if l.startswith('=='):
        p=l.split(); cur=(p[4],p[5],p[6].split('=')[1]); continue
    try: d=json.loads(l)
    except Exception: continue
    tab.setdefault((cur[0],cur[1],d['nq']),{})[cur[2]]=(d['call_ms'],d['kernel_ms'],d['parts'])
for k,v in tab.items(): print(k, v)
PY
