"""Top SASS instructions by warp-stall samples from `ncu -i X.ncu-rep --page source --csv`.
Usage: python tools/ncu_hot.py file.csv [top_n] [context]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
tot = sum(int(r[ix["# Samples"]] or 0) for r in body)
tot_inst = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
print(f"total samples {tot}, warp instructions executed {tot_inst}, SASS lines {len(body)}")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(int(r[ix[s]] or 0) for r in body) for s in stalls}
print("stall totals:", ", ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
order = sorted(range(len(body)), key=lambda i: -int(body[i][ix["# Samples"]] or 0))[:top]
for i in sorted(order):
    r = body[i]
    s = int(r[ix["# Samples"]] or 0)
    why = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:2]
    print(f"{i:5d} {s:7d} {100.0 * s / tot:5.1f}%  ex={r[ix['Instructions Executed']]:>9}  {r[ix['Source']].strip()[:90]:90s} {why}")
