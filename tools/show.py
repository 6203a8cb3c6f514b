#!/usr/bin/env python
"""Print steps/s and per-step event counts of bench JSON lines: tools/show.py FILES..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}
    e = r.get("events_per_launch", {})
    s = max(e.get("steps", 1), 1)
    ev = {k: round(v / s, 3) for k, v in e.items() if v and k != "steps"}
    print(f"{f}: {d['value']/1e9:.3f} G steps/s  {d['ms_per_step']:.2f} ms  graph {d.get('graph_device_bytes',0)/1e9:.2f} GB  {ev}")
