#!/usr/bin/env python
"""Summarise an ncu report (--set full) of the walk kernel into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep [--steps N] > profiles/rNN_X.md

Prints the counters DESIGN.md §7 reasons with: duration, DRAM bytes (read /
write) and throughput, L1/L2 sector hit rates, sectors per request, warp
stall samples, occupancy, divergence, registers.
"""
import argparse
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1)"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 write sectors (from L1)"),
    ("lts__t_sectors_srcunit_tex_lookup_miss.sum", "L2 lookup misses (from L1)"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (blocks, registers)"),
    ("launch__grid_size", "grid size"),
    ("launch__block_size", "block size"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps per cycle"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--steps", type=float, default=None, help="realised walk steps in the launch")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        print(f"## {a.title or a.rep}\n")
        print(f"kernel: `{d.get('Kernel Name', ('', '?'))[1][:160]}`\n")
        print("| counter | value | unit |\n|---|---|---|")
        for k, label in KEYS:
            if k in d:
                print(f"| {label} (`{k}`) | {d[k][1]} | {d[k][0]} |")
        stalls = sorted(((float(v[1].replace(",", "")), k) for k, v in d.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                         and v[1] not in ("", "n/a")), reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        print("\nwarp-state samples (top):\n")
        for s, k in stalls[:6]:
            print(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * s / tot:.1f}%")
        if a.steps:
            def num(k):
                u, v = d[k]
                x = float(v.replace(",", ""))
                return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)
            rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
            print(f"\nper realised step ({a.steps:.3g} steps): DRAM read {rd / a.steps:.1f} B, "
                  f"write {wr / a.steps:.1f} B, L2 read sectors "
                  f"{num('lts__t_sectors_srcunit_tex_op_read.sum') / a.steps:.1f}")
        print()


if __name__ == "__main__":
    main()
