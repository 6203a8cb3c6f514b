#!/usr/bin/env python
"""Per-source-line instruction / stall attribution from an ncu report (needs -lineinfo).
    python tools/ncu_lines.py gpurun_out/prof_X.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}; continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    try:
        ins = float(r[hdr["Instructions Executed"]].replace(",", ""))
        smp = float(r[hdr["Warp Stall Sampling (All Samples)"]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        continue
    k = (cur, int(r[0]))
    a = agg.get(k, [0.0, 0.0, r[1][:90]])
    a[0] += ins; a[1] += smp
    agg[k] = a
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti/1e9:.1f} G")
print(" inst%  stall%  file:line  source")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ti:5.1f} {100*v[1]/ts:6.1f}  {k[0]}:{k[1]}  {v[2]}")
