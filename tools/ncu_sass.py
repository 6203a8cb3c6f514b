#!/usr/bin/env python
"""SASS listing with per-instruction executed counts from an ncu source CSV
(--page source --csv --print-source cuda,sass), in address order:
    python tools/ncu_sass.py gpurun_out/X_src.csv.gz > listing.txt"""
import csv, gzip, io, sys
path = sys.argv[1]
raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
cur, hdr, line, rows = None, None, None, []
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = {}
        for i, h in enumerate(r):
            hdr.setdefault(h, i)
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        line = f"{cur}:{r[0]}"
        continue
    addr = r[2]
    if not addr.startswith("0x"):
        continue
    try:
        ins = float(r[hdr["Instructions Executed"]].replace(",", "") or 0)
        thr = float(r[hdr["Thread Instructions Executed"]].replace(",", "") or 0)
        smp = float(r[hdr["Warp Stall Sampling (All Samples)"]].replace(",", "") or 0)
    except (ValueError, KeyError):
        continue
    rows.append((int(addr, 16), ins, thr, smp, r[3].strip(), line))
rows.sort()
seen = set(); rows = [r for r in rows if not (r[0] in seen or seen.add(r[0]))]
tot = sum(x[1] for x in rows) or 1
b0 = rows[0][0] if rows else 0
for a, ins, thr, smp, sass, ln in rows:
    at = thr / ins if ins else 0
    print(f"{a - b0:6x} {100 * ins / tot:6.3f}% {at:5.1f} {int(smp):7d}  {sass:60s} {ln}")
