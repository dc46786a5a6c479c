#!/bin/bash
# Second A/B: queue kernel for every database that can seed its thresholds (XFBQ_UMMA_QUEUE_MIN_N=1), and shorter slices.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/queue_min_ab2_r2d.log
: > $O
for shape in "100000 128 10" "150000 128 10" "200000 256 100" "300000 256 100" "500000 256 100" "1000000 256 100" "1000000 128 1000" "2500000 256 100"; do
  for arm in "2000000 512" "1 512" "1 32"; do
    set -- $arm
    echo "== n dim k = $shape  arm=$1/$2" >> $O
    XFBQ_UMMA_QUEUE_MIN_N=$1 XFBQ_UMMA_MIN_SLICE=$2 timeout 600 python tools/batch_sweep.py $shape 32,100,256,1024,4096 >> $O 2>&1
  done
done
python - <<'PY'
import json
cur=None; tab={}
for l in open('gpurun_out/queue_min_ab2_r2d.log'):
    if l.startswith('=='):
        p=l.split(); cur=(p[5],p[6],p[7],p[8]); continue
    try: d=json.loads(l)
    except Exception: continue
    tab.setdefault((cur[0],cur[1],cur[2],d['nq']),{})[cur[3]]=(d['call_ms'],d['parts'])
for k,v in tab.items(): print(k, v)
PY
