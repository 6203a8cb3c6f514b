#!/usr/bin/env python
"""Compact an ncu launch list (--metrics gpu__time_duration.sum --csv) of one bench run:
every launch of the library's kernels in order, the framework / generator kernels
aggregated per name, and the walk kernel's share of all GPU time.

    python tools/launch_list.py gpurun_out/launches_X.csv > profiles/rNN_X_launches.csv"""
import csv, io, sys
from collections import OrderedDict

rows = [r for r in csv.reader(io.StringIO("".join(l for l in open(sys.argv[1]) if not l.startswith("=="))))]
hdr = {h: i for i, h in enumerate(rows[0])}
ours, other = [], OrderedDict()
LIB = ("walk_", "build_", "hash", "grape", "prefix", "validate", "guide", "record", "notri", "fence")
for r in rows[1:]:
    if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name, ns = r[hdr["Kernel Name"]], float(r[hdr["Metric Value"]])
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    if any(k in short for k in LIB):
        ours.append((r[hdr["ID"]], short, name.split(">(")[0][:160], r[hdr["Grid Size"]], r[hdr["Block Size"]], ns))
    else:
        c = other.setdefault(short[:100], [0, 0.0])
        c[0] += 1
        c[1] += ns
tot = sum(x[-1] for x in ours) + sum(v[1] for v in other.values())


def timed_walk(short):
    """walk kernels except the counting build (walk_tab_kernel's 6th template argument,
    STATS, launched once by bench.py outside the timed region for the roofline counts)"""
    if "walk_" not in short:
        return False
    if "walk_tab_kernel<" in short:
        return short.split("<")[1].rstrip(">").split(",")[5].strip() == "0"
    return True


walk = sum(x[-1] for x in ours if timed_walk(x[1]))
w = csv.writer(sys.stdout)
w.writerow(["# total GPU ns", int(tot), "walk-kernel ns", int(walk), "walk share", f"{walk / tot:.4f}"])
w.writerow(["ID", "kernel", "instance", "grid", "block", "duration_ns"])
for x in ours:
    w.writerow([x[0], x[1], x[2], x[3], x[4], int(x[5])])
w.writerow(["# other kernels (torch / generator), aggregated per name: count, total ns"])
for k, (c, ns) in sorted(other.items(), key=lambda kv: -kv[1][1]):
    w.writerow(["agg", k, c, "", "", int(ns)])
