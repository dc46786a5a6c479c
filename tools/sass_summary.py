"""Mnemonic counts of the shipped library's SASS (cuobjdump), per kernel family: the evidence that the hot path is tcgen05 /
TMA / tensor-memory code.  Usage: python tools/sass_summary.py > profiles/sass_summary_r2.txt"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = ROOT / "paper_2008_02002_b200" / "libxfbq_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
demangle = lambda n: subprocess.run(["cu++filt", n], capture_output=True, text=True).stdout.strip() or n
watch = ["UTCIMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "IMMA.16832.S8.U8", "POPC", "LOP3", "DFMA", "LDG.E.128", "ATOMS", "REDG", "ATOMG", "MATCH"]
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        op = m.group(1)
        per[cur]["_total"] += 1
        for w in watch:
            if op.startswith(w):
                per[cur][w] += 1
print(f"SASS summary of {lib.name} (sm_100a), {len(per)} kernels; counts of instruction mnemonics by prefix")
tot = collections.Counter()
for fn, c in per.items():
    tot.update(c)
print("whole library:", ", ".join(f"{w}={tot[w]}" for w in watch if tot[w]), f"(of {tot['_total']} instructions)")
print()
for fn, c in per.items():
    name = demangle(fn)
    name = name.replace("(int)", "").replace("(bool)", "")
    name = re.sub(r"\((?:const |unsigned |umma::|mma::|coop::|long|int|float|double|void).*", "", name)[:110]
    hits = ", ".join(f"{w}={c[w]}" for w in watch if c[w])
    print(f"{c['_total']:6d}  {name}\n        {hits}")
