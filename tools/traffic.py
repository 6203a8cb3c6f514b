#!/usr/bin/env python
"""Write profiles/traffic_cfgK.json (DRAM bytes per launch of the walk kernel) from
an ncu report of one timed launch:  tools/traffic.py REP K [mode [sampler]]
(sampler cdf: profiles/traffic_cfgK_cdf.json, read by bench.py --sampler cdf)"""
import csv, io, json, subprocess, sys
rep, k = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
vals = rows[2] if len(rows) > 2 else rows[1]
col = {h: i for i, h in enumerate(hdr)}
def get(name):
    return float(vals[col[name]].replace(",", ""))
unit_row = rows[1]
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rd *= scale.get(unit_row[col["dram__bytes_read.sum"]], 1)
wr *= scale.get(unit_row[col["dram__bytes_write.sum"]], 1)
kern = vals[col["Kernel Name"]]
mode = sys.argv[3] if len(sys.argv) > 3 else "node2vec"
out = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "kernel": kern,
       "source": rep.split("/")[-1], "mode": mode}
sampler = sys.argv[4] if len(sys.argv) > 4 else "rejection"
if sampler != "rejection":
    out["sampler"] = sampler
json.dump(out, open(f"profiles/traffic_cfg{k}{'' if sampler == 'rejection' else '_' + sampler}.json", "w"), indent=1)
print(json.dumps(out))
