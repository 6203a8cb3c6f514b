#!/usr/bin/env python
"""Summarise a reduced ncu capture (tools/profile_r02.sh: <rep>_raw.csv + <rep>_src.csv)
into markdown for profiles/:  python tools/ncu_csv_summary.py gpurun_out/prof_r02_cfg2 > profiles/X.md"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid size"),
    ("launch__block_size", "block size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps per cycle"),
]


def main():
    base = sys.argv[1]
    rows = list(csv.reader(open(base + "_raw.csv")))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"## {base.split('/')[-1]} (reduced on the box from the ncu --set full report)\n")
    print(f"kernel: `{vals[col['Kernel Name']]}`\n")
    print("| counter | value | unit |\n|---|---|---|")
    for k, name in KEYS:
        if k in col:
            print(f"| {name} (`{k}`) | {vals[col[k]]} | {units[col[k]]} |")
    st = []
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("\nwarp-state samples (top):\n")
    for v, h in sorted(st, reverse=True)[:8]:
        print(f"- {h}: {100 * v / tot:.1f}%")
    # SASS instruction mix (the source page of the report, per instruction)
    try:
        import collections
        import gzip
        src = list(csv.reader(open(base + "_src.csv")))
        h = src[1] if len(src[0]) < 4 else src[0]
        start = src.index(h) + 1
        ii = h.index("Instructions Executed")
        ti = h.index("Thread Instructions Executed")
        li = h.index("Source")
        op, opt = collections.Counter(), collections.Counter()
        for r in src[start:]:
            try:
                n, t = int(r[ii]), int(r[ti])
            except (ValueError, IndexError):
                continue
            f = r[li].split()
            o = f[1] if f and f[0].startswith("@") and len(f) > 1 else (f[0] if f else "?")
            o = o.split(".")[0]
            op[o] += n
            opt[o] += t
        tot = sum(op.values()) or 1
        print("\n### SASS instruction mix (share of warp instructions, average active threads)\n")
        print("| opcode | share | active threads |\n|---|---|---|")
        for o, n in op.most_common(16):
            print(f"| {o} | {100 * n / tot:.1f}% | {opt[o] / n:.1f} |")
    except (OSError, ValueError) as ex:
        print(f"\n(source page unavailable: {ex})")


if __name__ == "__main__":
    main()
