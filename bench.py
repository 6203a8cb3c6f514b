#!/usr/bin/env python
"""Benchmark: node2vec random-walk steps/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config 2] [--impl ours|reference]

One "step" of this benchmark = one pass of the whole hot path over one batch:
grape_walks_node2vec over every walk of the workload (BASELINE configs[1] by
default: Chung-Lu 1M nodes / ~20M edges, weights U{1..100}, p=0.5, q=2,
10 walks per node, L=80).  N > 1 (torchrun): every rank holds a replica of
the graph (BASELINE north_star: "replicated on every GPU ... walks sharded by
start node") and walks its contiguous slice [floor(r W/N), floor((r+1) W/N)) of
the config's fixed, iteration-major walk list with walk_id_base = the slice
start (--scaling strong, the default: the same total work at every N, so the
concatenated rank matrices are the N = 1 matrix bit for bit).  --scaling weak
gives every rank the whole per-GPU workload on its own wid block instead.
No collective is on the data path.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (the only reference this paper-tier
task has) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from graphgen import CONFIGS, config_graph, config_walks, starts_per_node  # noqa: E402


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,clocks.mem,temperature.gpu,temperature.memory")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's NVML start-up can stall the GPU (measured: one launch of a timed
            # region took 214 ms instead of 47): wait for its first sample, i.e. until it is
            # up and polling, before the timed region starts
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 10.0:
                time.sleep(0.02)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, mem, tg, tm = [], 0.0, set(), [], [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
            for lst, k in ((mem, 7), (tg, 8), (tm, 9)):
                try:
                    lst.append(float(parts[k]))
                except (ValueError, IndexError):
                    pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        med = lambda v: float(np.median(v)) if v else None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "mem_mhz": med(mem), "gpu_temp_c": med(tg), "mem_temp_c": med(tm)}


def _dist_setup(args):
    """(world, rank, device index).  The device is LOCAL_RANK unless --device pins every
    rank to one GPU (the two-process parity test: both ranks on cuda:0, which needs the
    gloo backend — NCCL refuses two ranks on one device)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.device is not None:
        local = args.device
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = args.dist_backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def _red_device(dev):
    """Where the small reduction tensors live: the GPU for NCCL, the host for gloo."""
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return torch.device("cpu")
    return dev


def rank_slice(W_total: int, per_gpu: int, rank: int, world: int, scaling: str):
    """(lo, hi) of the iteration-major wid list this rank walks.
    strong: the config's W_total walks split into contiguous start-node slices;
    weak: per_gpu walks per rank on wid block [r per_gpu, (r+1) per_gpu)."""
    from paper_2110_06196_b200.shard import shard_range, weak_scaling_range
    if scaling == "strong":
        return shard_range(W_total, rank, world)
    return weak_scaling_range(per_gpu, rank, world)


def _allreduce(x: float, op, world):
    if world == 1:
        return x
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() != "gloo" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def _allgather(x: float, world):
    if world == 1:
        return [x]
    out = [None] * world
    dist.all_gather_object(out, float(x))
    return out


def _oracle_sample(g_cpu, wk, budget_s: float, first_wid: int = 0, cores: int | None = None, dT: int = 0,
                   sampler: str = "rejection"):
    """Run the oracle (as it stands) on consecutive walks until ~budget_s of CPU
    work per thread; returns (realised steps, seconds, walks, threads, attempts).
    sampler: the node2vec rule the GPU arm runs (rejection / cdf / folded)."""
    from oracle.oracle import Oracle
    o = Oracle(*g_cpu.numpy())
    if wk["mode"] == "node2vec" and not dT and sampler in ("cdf", "folded"):
        alt = o.walks_cdf if sampler == "cdf" else o.walks_folded

        class _O:   # the same call shape as Oracle.walks for the sampling loop below
            @staticmethod
            def walks(starts, L, mode, p, q, seed, base=0, with_attempts=False):
                out, st = alt(starts, L, p=p, q=q, seed=seed, base=base)
                return (out, st, 0) if with_attempts else (out, st)
        o = _O()
    n = g_cpu.n
    cores = cores or os.cpu_count() or 1
    W = n * wk["walks_per_node"]
    starts_all = (np.arange(W, dtype=np.int64) % n).astype(np.uint32)
    # calibrate the per-thread batch on 64 walks
    t0 = time.perf_counter()
    if dT:
        _, s0 = o.walks_approx(starts_all[:64], wk["L"], dT, mode=wk["mode"], p=wk["p"], q=wk["q"], seed=wk["seed"])
    else:
        _, s0 = o.walks(starts_all[:64], wk["L"], mode=wk["mode"], p=wk["p"], q=wk["q"], seed=wk["seed"])
    dt = max(time.perf_counter() - t0, 1e-4)
    per_thread = max(64, int(64 * budget_s / dt))
    total = min(W - first_wid, per_thread * cores)
    chunks = np.array_split(np.arange(first_wid, first_wid + total), cores)
    res = [None] * cores

    def work(k):
        ids = chunks[k]
        if len(ids) == 0:
            res[k] = (0, 0)
            return
        if dT:
            _, st = o.walks_approx(starts_all[ids[0]:ids[-1] + 1], wk["L"], dT, mode=wk["mode"], p=wk["p"],
                                   q=wk["q"], seed=wk["seed"], base=int(ids[0]))
            att = 0
        else:
            _, st, att = o.walks(starts_all[ids[0]:ids[-1] + 1], wk["L"], mode=wk["mode"], p=wk["p"],
                                 q=wk["q"], seed=wk["seed"], base=int(ids[0]), with_attempts=True)
        res[k] = (st, att)

    th = [threading.Thread(target=work, args=(k,)) for k in range(cores)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    secs = time.perf_counter() - t0
    steps = sum(r[0] for r in res)
    att = sum(r[1] for r in res)
    return steps, secs, int(total), cores, att


L2_BYTES = 126 * 2 ** 20
FLUSH_BYTES = 512 * 2 ** 20


def _cpu_model() -> str:
    """The host CPU's model name (lscpu), for the cpu_baseline record."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def _gpu_local_cpus(local):
    """The CPUs next to GPU `local` (its PCI device's local_cpulist in sysfs) that this
    process may run on; None when unknown."""
    try:
        pr = torch.cuda.get_device_properties(local)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def _cpu_ranges(cpus):
    xs = sorted(cpus)
    out, a = [], xs[0]
    for p_, q_ in zip(xs, xs[1:] + [None]):
        if q_ != p_ + 1:
            out.append(f"{a}-{p_}" if p_ != a else f"{a}")
            a = q_
    return ",".join(out)


def _dram_probe(launch, dev):
    """DRAM bytes (read + write) of the kernels `launch` runs, from the GPU counters
    (tools/libgrape_dram_probe.so, CUPTI range profiler; untimed).  None if unavailable."""
    path = os.path.join(ROOT, "tools", "libgrape_dram_probe.so")
    if not os.path.exists(path):
        return None
    try:
        import ctypes
        lib = ctypes.CDLL(path)
        lib.grape_dram_probe_error.restype = ctypes.c_char_p
        torch.cuda.synchronize(dev)
        if lib.grape_dram_probe_begin() != 0:
            print("dram probe:", lib.grape_dram_probe_error().decode(), file=sys.stderr)
            return None
        launch()
        torch.cuda.synchronize(dev)
        rd, wr, ns = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        if lib.grape_dram_probe_end(ctypes.byref(rd), ctypes.byref(wr), ctypes.byref(ns)) != 0:
            print("dram probe:", lib.grape_dram_probe_error().decode(), file=sys.stderr)
            return None
        return rd.value + wr.value if rd.value + wr.value > 0 else None
    except Exception as ex:   # measurement aid only: never fail the bench over it
        print("dram probe:", ex, file=sys.stderr)
        return None


def _issue_probe(launch, dev):
    """Issue counters of the kernels `launch` runs (one more untimed launch; the probe's metric
    set 1): warp instructions, thread instructions, cycles with an instruction issued and active
    cycles, each summed over the SM sub-partitions.  None if unavailable."""
    path = os.path.join(ROOT, "tools", "libgrape_dram_probe.so")
    if not os.path.exists(path):
        return None
    try:
        import ctypes
        lib = ctypes.CDLL(path)
        lib.grape_dram_probe_error.restype = ctypes.c_char_p
        if not hasattr(lib, "grape_probe_begin_set"):
            return None
        torch.cuda.synchronize(dev)
        if lib.grape_probe_begin_set(1) != 0:
            print("issue probe:", lib.grape_dram_probe_error().decode(), file=sys.stderr)
            return None
        launch()
        torch.cuda.synchronize(dev)
        v = (ctypes.c_double * 4)()
        if lib.grape_probe_end_set(v) != 0:
            print("issue probe:", lib.grape_dram_probe_error().decode(), file=sys.stderr)
            return None
        if v[0] <= 0 or v[3] <= 0:
            return None
        return {"warp_instructions": v[0], "thread_instructions": v[1], "issue_active_cycles": v[2],
                "active_cycles": v[3]}
    except Exception as ex:   # measurement aid only: never fail the bench over it
        print("issue probe:", ex, file=sys.stderr)
        return None


def _needs_flush(g, W, L):
    """Workloads whose CSR and output fit twice in L2 get an L2 flush between timed steps
    (decided from the CSR, so both arms state the same config)."""
    csr = 8 * (g.n + 1) + 4 * g.m * (2 if g.w is not None else 1)
    return csr + 4 * W * L < 2 * L2_BYTES


def _workload_desc(k, g, wk, W, flush=False):
    wl = (f"BASELINE configs[{k - 1}]: {CONFIGS[k]['name']}" if k <= 5 else
          f"beyond BASELINE (index-range demonstration): {CONFIGS[k]['name']}")
    return {"workload": wl, "mode": wk["mode"], "graph": g.name,
            "nodes": g.n, "arcs": g.m, "weighted": g.w is not None, "walks_per_gpu": W, "L": wk["L"],
            "p": wk["p"], "q": wk["q"], "seed": wk["seed"],
            "l2": ("flushed: a 512 MB buffer is written between timed steps (graph + output fit in the 126 MB L2)"
                   if flush else "no flush: per-step output (W*L*4 B) and graph exceed the 126 MB L2")}


def run_reference(args):
    # CPU only: no process group (rank 0 alone runs and prints; the others exit 0)
    if int(os.environ.get("RANK", "0")) != 0:
        return
    k = args.config
    wk = _walk_recipe(args)
    g = config_graph(k)
    W = g.n * wk["walks_per_node"]
    vals, total_steps, total_secs = [], 0, 0.0
    for i in range(args.warmup + args.steps):
        steps, secs, walks, cores, _ = _oracle_sample(g, wk, args.ref_budget, first_wid=(i * 997) % max(W - 1, 1),
                                                      dT=args.approx, sampler=args.sampler)
        if i >= args.warmup:
            vals.append(steps / secs)
            total_steps += steps
            total_secs += secs
    v = total_steps / total_secs
    metric = ("random-walk steps/sec (node2vec 2nd-order)" if wk["mode"] == "node2vec" else
              "random-walk steps/sec (first-order)")
    if args.approx:
        metric = metric[:-1] + f", approximated: SUSS d_T={args.approx})"
    if wk["mode"] == "node2vec" and args.sampler == "cdf":
        metric = metric[:-1] + ", paper CDF sampler)"
    if wk["mode"] == "node2vec" and args.sampler == "folded":
        metric = metric[:-1] + ", outlier-folded rejection)"
    line = {"impl": "reference", "metric": metric, "value": v,
            "unit": "steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_secs / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u32/u64 integer", "data": "synthetic (seeded generator)",
            "config": _workload_desc(k, g, wk, W, _needs_flush(g, W, wk["L"])),
            "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"{walks} consecutive walks per step of the workload (bounded sample)"},
            "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _parse_layout(spec: str):
    if not spec:
        return None
    return {k: int(float(v)) for k, v in (kv.split("=") for kv in spec.split(","))}


def _walk_recipe(args):
    wk = config_walks(args.config)
    if args.mode:
        wk["mode"] = args.mode
    return wk


def run_ours(args):
    world, rank, local = _dist_setup(args)
    import paper_2110_06196_b200 as grape
    from paper_2110_06196_b200.shard import reduce_step_timing
    k = args.config
    wk = _walk_recipe(args)
    dev = torch.device("cuda", local)
    g = config_graph(k, device=dev, scale_down=args.scale_down)
    torch.cuda.empty_cache()   # the generator's temporaries: room for the graph's tables
    # a1 graph build (validation, prefix, node records, sampling tables): synchronous
    # C-ABI call, timed on its own (outside the timed walk region, reported).  A tiny graph
    # is built first so the one-time loading of the library's kernels into the context
    # (CUDA lazy module loading: ~0.6 s on the first build of a process) is not counted.
    from graphgen import tiny_graph
    _t = tiny_graph(1, 40, 0.1, weighted=g.w is not None)
    grape.graph_from_csr(_t.off, _t.col, _t.w, device=local, symmetric=True).free()
    del _t
    torch.cuda.synchronize(dev)
    t_b = time.perf_counter()
    if args.dist_tables:   # §8(f) f4: part r of the tables on rank r, built by all ranks together
        if world < 2:
            raise SystemExit("--dist-tables needs N > 1 ranks (torchrun)")
        dg = grape.graph_from_csr_dist(g.off, g.col, g.w, device=local, symmetric=g.symmetric,
                                       layout=_parse_layout(args.layout),
                                       table_budget_bytes=int(args.table_budget * 1e9) if args.table_budget else None)
    else:
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=local, symmetric=g.symmetric, tables=not args.no_tables,
                                  layout=_parse_layout(args.layout))
    torch.cuda.synchronize(dev)
    build_ms = 1e3 * (time.perf_counter() - t_b)
    g = g.to("cpu")            # the library holds its own copy; free the device CSR for the walk matrix
    torch.cuda.empty_cache()
    if args.parts > 1:         # §8(f) f4 layout: tables in power-of-two parts (on this GPU)
        dg.partition([local] * args.parts)
    info = dg.info
    W_total = g.n * wk["walks_per_node"]          # the config's walk list (iteration-major)
    if args.max_walks:                            # profiling runs: the first walks of the list only
        W_total = min(W_total, args.max_walks)
    L = wk["L"]
    lo, hi = rank_slice(W_total, W_total, rank, world, args.scaling)
    if args.slice:   # one rank's slice of an N-rank strong-scaling run, walked by this single process
        r_, n_ = (int(t) for t in args.slice.split("/"))
        if world > 1 or not 0 <= r_ < n_ or args.scaling != "strong":
            raise SystemExit("--slice R/N: one process, 0 <= R < N, strong scaling")
        lo, hi = rank_slice(W_total, W_total, r_, n_, "strong")
    base = lo
    W = hi - lo                                   # this rank's walks
    if args.scaling == "strong":
        starts = starts_per_node(g.n, wk["walks_per_node"], device=dev)[lo:hi].contiguous()
    else:
        starts = starts_per_node(g.n, wk["walks_per_node"], device=dev)[:W].contiguous()
    out = torch.empty((W, L), dtype=torch.int32, device=dev)
    steps_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    node2vec = wk["mode"] == "node2vec"

    dT = args.approx

    def call(st_buf, out_buf, ctr):
        kw = dict(seed=wk["seed"], walk_id_base=base, out=out_buf, steps=ctr)
        if dT:
            grape.walks_approx(dg, st_buf, L, dT, node2vec=node2vec, p=wk["p"], q=wk["q"], **kw)
        elif args.sampler == "cdf":
            grape.walks_node2vec_cdf(dg, st_buf, L, wk["p"], wk["q"], **kw)
        elif args.sampler == "folded" and node2vec:
            grape.walks_node2vec_folded(dg, st_buf, L, wk["p"], wk["q"], **kw)
        elif node2vec:
            grape.walks_node2vec(dg, st_buf, L, wk["p"], wk["q"], **kw)
        else:
            grape.walks_first_order(dg, st_buf, L, **kw)

    def one(ctr):
        call(starts, out, ctr)

    for _ in range(args.warmup):
        one(None)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    flush = _needs_flush(g, W, L)
    scrub = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev) if flush else None
    with ClockSampler(local) as clk:
        # ~100 ms of GPU spin queued ahead of the first start event: the host enqueues the
        # timed launches while the GPU is busy, so a host-side pause (measured: sporadic
        # 20-170 ms pauses of the host on these boxes) cannot open an idle gap between a
        # start event and its launch — the events measure the kernels, not the host
        torch.cuda._sleep(int(0.1 * 1.9e9))
        t_wall = time.perf_counter()
        for i in range(args.steps):
            if flush:
                scrub.fill_(i)   # evicts the graph and the previous output from L2 (untimed)
            ev[i][0].record(stream)
            one(steps_ctr)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = float(sum(kernel_ms))
    my_steps = float(steps_ctr.item())
    max_ms, tot_steps = reduce_step_timing(my_ms, my_steps, world, device=_red_device(dev))
    rank_ms = _allgather(my_ms / args.steps, world)     # per-rank ms per step (tail imbalance)
    if args.dump_walks:   # the rank's walk matrix, for the multi-process parity test
        np.save(f"{args.dump_walks}.rank{rank}.npy", out.cpu().numpy().view(np.uint32))
        with open(f"{args.dump_walks}.rank{rank}.json", "w") as f:
            json.dump({"lo": lo, "hi": hi, "steps": my_steps / args.steps}, f)
    value = tot_steps / (max_ms / 1e3)
    steps_per_launch = my_steps / args.steps
    avg_launch_ms = my_ms / args.steps

    # ---- e2e: same metric through the C-ABI with HOST buffers (pinned), H2D/D2H inside
    e2e = None
    h_out = None
    host_cpus = None
    if not args.no_e2e:
        # the pinned buffers are first-touched from the CPUs next to the GPU (its PCI
        # device's local_cpulist), so on a multi-socket host their pages sit on the GPU's
        # NUMA node and the copies do not cross the socket link; the thread's affinity is
        # restored after.  (The pool's boxes have one NUMA node: a no-op there, measured
        # equal; their occasional slow host-buffer calls are host-side pauses.)
        host_cpus = None if os.environ.get("GRAPE_BENCH_NUMA") == "0" else _gpu_local_cpus(local)   # (A/B knob)
        saved = os.sched_getaffinity(0) if host_cpus else None
        if host_cpus:
            os.sched_setaffinity(0, host_cpus)
        try:
            h_starts = starts.cpu().pin_memory()
            try:   # W*L*4 bytes of pinned host memory per rank (34 GB on configs[4])
                h_out = torch.empty((W, L), dtype=torch.int32, pin_memory=True)
            except RuntimeError as ex:
                e2e = {"unavailable": f"pinned host buffer of {W * L * 4 / 1e9:.1f} GB: {str(ex)[:120]}"}
        finally:
            if saved:
                os.sched_setaffinity(0, saved)
        if _allreduce(1.0 if h_out is not None else 0.0, dist.ReduceOp.MIN, world) < 1.0:
            h_out = None   # every rank skips together (no half-entered collective)
            e2e = e2e or {"unavailable": "a rank could not pin its host buffer"}
    e2e_one_ms = None
    if h_out is not None:
        h_steps = torch.zeros(1, dtype=torch.int64)
        time.sleep(1.0)            # the clock sampler's nvidia-smi has just exited (its NVML teardown)
        # warm-up of the host path, as many calls as the device warm-up (at least 2): the first
        # calls on a freshly pinned multi-GB buffer ran 450-730 ms instead of 65 ms on a box
        # whose host memory a previous process had just used
        for _ in range(max(2, args.warmup)):
            call(h_starts, h_out, None)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e2e_steps = args.steps   # the same K steps as the device-timed region
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            t1 = time.perf_counter()
            call(h_starts, h_out, h_steps)
            print(f"e2e call {1e3 * (time.perf_counter() - t1):.1f} ms", file=sys.stderr, flush=True)
        torch.cuda.synchronize(dev)
        e2e_s = time.perf_counter() - t0
        e2e_s = _allreduce(e2e_s, dist.ReduceOp.MAX, world)
        e2e_one_ms = 1e3 * e2e_s / e2e_steps
        e2e_tot = _allreduce(float(h_steps.item()), dist.ReduceOp.SUM, world)
        e2e = {"value": e2e_tot / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": int(W * 4),
               "d2h_bytes_per_step": int(W * L * 4 + 8), "steps_timed": e2e_steps,
               "host_buffers": ("pinned, first-touched on the GPU-local CPUs " + _cpu_ranges(host_cpus)
                                if host_cpus else "pinned (GPU-local CPUs unknown)"),
               "path": ("grape_walks_approx" if dT else
                        ("grape_walks_node2vec_cdf" if args.sampler == "cdf" else
                         "grape_walks_node2vec_folded" if args.sampler == "folded" else
                         "grape_walks_node2vec") if node2vec else "grape_walks_first_order") +
                       " with pinned host starts/out (library-staged, chunked H2D/kernel/D2H)"}

    build_max = _allreduce(build_ms, dist.ReduceOp.MAX, world)   # every rank builds its replica
    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        s, secs, walks, cores, att = _oracle_sample(g, wk, args.cpu_budget, dT=dT, sampler=args.sampler)
        s1, secs1, walks1, _, _ = _oracle_sample(g, wk, max(1.0, args.cpu_budget / 4), dT=dT, sampler=args.sampler,
                                                 cores=1)
        cpu = {"value": s / secs, "unit": "steps/s", "cores": cores, "kind": "oracle",
               "cpu_model": _cpu_model(),
               "single_thread": {"value": s1 / secs1, "unit": "steps/s", "walks": walks1,
                                 "seconds": round(secs1, 2)},
               "sample": f"first {walks} walks (wid 0..{walks - 1}) of the same workload, "
                         f"{cores} threads, {secs:.1f} s; single thread: first {walks1} walks, {secs1:.1f} s"}
    # ---- roofline of the walk kernel: event counts from the counting
    # build of the same kernel (grape_walks_stats, untimed), times the measured time.
    roof = None
    issue_raw = None
    if rank == 0 and args.sampler != "cdf":   # (no counting build of the CDF sampler)
        _, ev = grape.walks_stats(dg, starts, L, node2vec=node2vec, p=wk["p"], q=wk["q"], seed=wk["seed"],
                                  degree_threshold=dT, sampler=args.sampler if node2vec else "rejection",
                                  walk_id_base=base, out=out)
        torch.cuda.synchronize(dev)
        weighted = info["cw_bytes"] > 0
        if info.get("tables"):
            # table walker: every read is one random 32-B sector that the
            # rules force given the tables — the node record of a start, one guide entry
            # or record per proposal whose x matters, the record of a taken arc, one
            # edge-hash bucket per membership probe; attempts decided from registers
            # read nothing.  (starts are read sequentially; counted as sectors too.)
            rand_sectors = ev["sector_loads"]
        else:
            # fenced-search walker: one sector per node record, one col sector per
            # proposal (+ one prefix leaf if weighted), one N(t) leaf per membership test
            rand_sectors = ev["node_loads"] + ev["attempts"] * (2 if weighted else 1) + ev["membership_tests"]
        alg_bytes = 32 * rand_sectors + 4 * W * L + 4 * W
        t_launch = avg_launch_ms / 1e3
        peak, peak_src = _peaks()
        traffic = args.traffic_per_launch
        traffic_src = "--traffic-per-launch" if traffic is not None else None
        if traffic is None and not args.no_probe:
            # DRAM bytes of one more (untimed) launch of the same call, read from the GPU's
            # counters in this run (tools/dram_probe.cpp, CUPTI range profiler)
            traffic = _dram_probe(lambda: one(None), dev)
            if traffic is not None:
                traffic_src = "measured in this run: CUPTI range profiler over one untimed launch (tools/dram_probe.cpp)"
                issue_raw = _issue_probe(lambda: one(None), dev)   # the issue counters of one more
        tfile = os.path.join(ROOT, "profiles", f"traffic_cfg{k}.json")
        kname = "walk_tab_kernel" if info.get("tables") else "walk_sm_kernel"
        if traffic is None and os.path.exists(tfile):
            tj = json.load(open(tfile))
            # only a capture of the same kernel and walk mode counts
            if (kname in tj.get("kernel", "") and tj.get("mode", wk["mode"]) == wk["mode"]
                    and tj.get("sampler", "rejection") == args.sampler and tj.get("dT", 0) == dT):
                traffic = tj["dram_bytes_per_launch"]
                traffic_src = f"profiles/traffic_cfg{k}.json (an earlier ncu capture of the same kernel)"
        # random-sector ceiling at this graph's randomly read footprint (measured,
        # profiles/gather_footprint.json; linear interpolation in footprint)
        ceil, ceil_src = None, None
        cfile = os.path.join(ROOT, "profiles", "gather_footprint.json")
        if os.path.exists(cfile):
            tab = json.load(open(cfile))["footprint_gb_vs_rate"]
            fp = info["device_bytes"] / 1e9
            xs, ys = [t[0] for t in tab], [t[1] for t in tab]
            if fp <= xs[0]:
                rate = ys[0]
            elif fp >= xs[-1]:
                rate = ys[-1]
            else:
                k_ = next(j for j in range(1, len(xs)) if xs[j] >= fp)
                rate = ys[k_ - 1] + (ys[k_] - ys[k_ - 1]) * (fp - xs[k_ - 1]) / (xs[k_] - xs[k_ - 1])
            ceil = rate * 1e9
            ceil_src = f"profiles/gather_footprint.json at {fp:.1f} GB"
        achieved = alg_bytes / t_launch / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": ("walk_tab_kernel" if info.get("tables") else "walk_sm_kernel") +
                          (" (grape_walks_node2vec)" if node2vec else " (grape_walks_first_order)"),
                "peak_source": peak_src, "avg_launch_ms": avg_launch_ms,
                "algorithmic_bytes_per_launch": alg_bytes,
                "bytes_per_step": alg_bytes / max(ev["steps"], 1),
                "events_per_launch": ev,
                # achieved HBM bandwidth (BASELINE metric): the ncu-measured DRAM bytes of one launch
                # of this kernel (profiles/traffic_cfgK.json) over the launch time measured here
                "dram_gbs": (traffic / t_launch / 1e9) if traffic else None,
                "dram_frac": (traffic / t_launch / 1e9 / peak) if traffic else None,
                "random_access": {"compulsory_sectors_per_step": rand_sectors / max(ev["steps"], 1),
                                  "achieved_per_s": rand_sectors / t_launch,
                                  "ceiling_per_s": ceil,
                                  "frac": (rand_sectors / t_launch / ceil) if ceil else None,
                                  "ceiling_source": ceil_src,
                                  "note": "the ceiling is the uniform-random dependent-read microbenchmark at this "
                                          "footprint (tools/gather_footprint.cu); reads with DRAM-page locality "
                                          "(records of one row, guide -> record) can exceed it"}}
    if rank == 0 and args.sampler == "cdf" and node2vec:
        # The CDF sampler has no counting build: its compulsory reads follow from the walks
        # themselves.  Step s >= 2 at v reads v's whole row of arc records (pass 1; pass 2
        # rescans one chunk of <= 32 records from L1/L2); the first step reads one record
        # and one guide entry or record.  Membership probes are not counted (a lower bound).
        deg = torch.diff(g.off.to(dev)).to(torch.int64)
        rb = int(info.get("record_bytes") or 32)
        row_bytes, first = 0.0, 0.0
        for r0 in range(0, W, 1 << 20):                      # row chunks: bounded temporaries
            blk = out[r0:r0 + (1 << 20)]
            vs = blk[:, 1:L - 1]                             # v of every step s >= 2
            live = (vs != -1) & (blk[:, 2:L] != -1)
            row_bytes += float((deg[vs[live].long()] * rb).sum().item())
            first += float((blk[:, 1] != -1).sum().item()) * 64
        alg_bytes = row_bytes + first + 4 * W * L + 4 * W
        t_launch = avg_launch_ms / 1e3
        peak, peak_src = _peaks()
        tfile = os.path.join(ROOT, "profiles", f"traffic_cfg{k}_cdf.json")
        traffic = None if args.no_probe else _dram_probe(lambda: one(None), dev)
        traffic_src = "measured in this run: CUPTI range profiler over one untimed launch (tools/dram_probe.cpp)"
        if traffic is None and os.path.exists(tfile):
            traffic = json.load(open(tfile))["dram_bytes_per_launch"]
            traffic_src = f"profiles/traffic_cfg{k}_cdf.json (an earlier ncu capture of the same kernel)"
        roof = {"bound": "hbm", "achieved": alg_bytes / t_launch / 1e9, "peak": peak, "unit": "GB/s",
                "frac": alg_bytes / t_launch / 1e9 / peak, "traffic": traffic, "traffic_source": traffic_src,
                "dram_gbs": (traffic / t_launch / 1e9) if traffic else None,
                "dram_frac": (traffic / t_launch / 1e9 / peak) if traffic else None,
                "kernel": "walk_cdf_kernel (grape_walks_node2vec_cdf)", "peak_source": peak_src,
                "avg_launch_ms": avg_launch_ms, "algorithmic_bytes_per_launch": alg_bytes,
                "bytes_per_step": alg_bytes / max(steps_per_launch, 1),
                "note": "bytes the paper's O(deg v) step touches, from the walk matrix: v's full row of "
                        "records per node2vec step, membership probes not counted; hub rows are largely "
                        "L2-resident, so DRAM traffic (dram_gbs) is below this"}
        del deg
    clocks = clk.summary()
    if rank == 0 and issue_raw and roof:
        # the instruction-issue side of the same launch: the walker's other bound.
        # Peak = one warp instruction per scheduler per cycle: SMs x 4 schedulers x the SM clock
        # sampled under load.
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz")
        t_l = roof["avg_launch_ms"] / 1e3
        wi = issue_raw["warp_instructions"]
        roof["issue"] = {
            "warp_instructions_per_launch": wi,
            "warp_instructions_per_step": wi / max(steps_per_launch, 1),
            "active_threads_per_instruction": issue_raw["thread_instructions"] / wi,
            "issue_active_frac": issue_raw["issue_active_cycles"] / issue_raw["active_cycles"],
            "achieved_per_s": wi / t_l,
            "peak_per_s": (sms * 4 * mhz * 1e6) if mhz else None,
            "frac": (wi / t_l / (sms * 4 * mhz * 1e6)) if mhz else None,
            "source": "measured in this run: CUPTI range profiler over one untimed launch (smsp__inst_executed, "
                      "smsp__thread_inst_executed, smsp__issue_active, smsp__cycles_active; tools/dram_probe.cpp); "
                      "peak = SMs x 4 schedulers x 1 warp instruction per cycle x the sampled SM clock"}
        # the utilisations side by side: the highest names what the launch is closest to being bound by
        fr = {"dram_traffic": roof.get("dram_frac"), "random_access": (roof.get("random_access") or {}).get("frac"),
              "issue": roof["issue"]["frac"]}
        fr = {k_: v_ for k_, v_ in fr.items() if v_ is not None}
        roof["utilisation"] = dict(fr, highest=max(fr, key=fr.get))
    if rank == 0:
        metric = "random-walk steps/sec (node2vec 2nd-order)" if node2vec else "random-walk steps/sec (first-order)"
        if dT:
            metric = metric[:-1] + f", approximated: SUSS d_T={dT})"
        if args.sampler == "cdf":
            metric = metric[:-1] + ", paper CDF sampler)"
        if args.sampler == "folded" and node2vec:
            metric = metric[:-1] + ", outlier-folded rejection)"
        if args.parts > 1:
            metric = metric[:-1] + f", tables in {args.parts} parts)"
        if args.dist_tables:
            metric = metric[:-1] + f", tables distributed over {world} GPUs)"
        cfg = _workload_desc(k, g, wk, W, flush)
        cfg.update({"walks_total": W_total if args.scaling == "strong" else W * world,
                    "sharding": ("strong: rank r walks wids [floor(r W/N), floor((r+1) W/N)) of the config's "
                                 "fixed list, walk_id_base = slice start (graph replicated)"
                                 if args.scaling == "strong" else
                                 "weak: every rank walks W wids on its own block [r W, (r+1) W)")})
        if args.scale_down:
            cfg["scale_down"] = args.scale_down
        if args.max_walks:
            cfg["max_walks"] = args.max_walks
        if args.slice:
            cfg["slice"] = f"{args.slice}: wids [{lo}, {hi}) only (one rank of an N-rank run, emulated on one GPU)"
        if args.dist_tables:
            cfg["tables"] = (f"distributed: rank r owns part r of the sampling tables ({world} parts, CUDA IPC), "
                             f"every rank walks over all parts")
        line = {"metric": metric, "value": value, "unit": "steps/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u32/u64 integer",
                "data": "synthetic (seeded generator, graphgen/)", "config": cfg,
                "rank_ms_per_step": [round(x, 3) for x in rank_ms],
                "rank_spread": (max(rank_ms) / min(rank_ms) - 1.0) if min(rank_ms) > 0 else None,
                "graph_build_ms": build_max,
                "one_pass": {"graph_build_ms": build_max, "walk_ms": max_ms / args.steps,
                             "e2e_walk_ms": e2e_one_ms,
                             "steps_per_s_incl_build": tot_steps / args.steps /
                                                       ((build_max + (e2e_one_ms or max_ms / args.steps)) / 1e3),
                             "note": "one pass from a device CSR: build the graph (validation, prefix, tables), "
                                     "then one walk call (host buffers when e2e ran)"},
                "gpu_launches": args.steps, "realised_steps_per_gpu_step": steps_per_launch,
                "step_ms": [round(x, 3) for x in kernel_ms],
                "nominal_steps_per_gpu_step": W * (L - 1), "wall_s_timed": t_wall,
                "clocks": clocks, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "graph_device_bytes": info["device_bytes"],
                "graph_layout": {k_: info.get(k_) for k_ in ("tables", "record_bytes", "guide_bytes", "guide_factor",
                                                              "hash_h", "notri", "weights_symmetric",
                                                              "table_bytes", "parts")}}
        print(json.dumps(line), flush=True)
    dg.free()
    if world > 1:
        dist.destroy_process_group()


def _sg_lookup_roofline(n, m, lookups, launch_s):
    """The pair kernel's bound: one random node-guide read per negative (rank of a
    uniform arc index) against the measured random-lookup rate at the
    guide's size (profiles/r02_l2_lookup.json, tools/l2_lookup.cu; log-size interpolation).
    The guide's size follows skipgram.cu ensure_node_guide: 16-B entries, 4 buckets
    per node while n * 64 B <= 128 MiB, else 1."""
    per_node = 4 if n * 64 <= (128 << 20) else 1
    sh = 0
    while (m >> sh) + 1 > per_node * n:
        sh += 1
    table = ((m >> sh) + 1) * 16
    try:
        ref = json.load(open(os.path.join(ROOT, "profiles", "r02_l2_lookup.json")))
    except OSError:
        return None
    mb = table / 2**20
    xs, ys = ref["table_mb"], ref["unroll1"]
    if mb <= xs[0]:
        ceil = ys[0]
    elif mb >= xs[-1]:
        ceil = ys[-1]
    else:
        j = next(i for i in range(1, len(xs)) if xs[i] >= mb)
        f = (math.log(mb) - math.log(xs[j - 1])) / (math.log(xs[j]) - math.log(xs[j - 1]))
        ceil = ys[j - 1] + f * (ys[j] - ys[j - 1])
    ach = lookups / launch_s / 1e9
    return {"lookups_per_launch": lookups, "achieved_G_per_s": ach, "ceiling_G_per_s": ceil, "frac": ach / ceil,
            "node_guide_bytes": table,
            "ceiling_source": "profiles/r02_l2_lookup.json (random 8-B lookups vs table size, this GPU model)"}


def run_skipgram(args):
    """--skipgram: the SkipGram consumer.  One step =
    the config's walks for a batch of B walk ids (the walk kernel) + their window-w
    pairs and K scale-free negatives (grape_skipgram_pairs), both on the device.
    Reports training slots/s of the whole step, the pair kernel alone, and the pair
    kernel's HBM roofline (its output words are written once, coalesced)."""
    world, rank, local = _dist_setup(args)
    import paper_2110_06196_b200 as grape
    from paper_2110_06196_b200.shard import weak_scaling_range
    k = args.config
    wk = _walk_recipe(args)
    win, K = args.window, args.negatives
    dev = torch.device("cuda", local)
    g = config_graph(k, device=dev)
    torch.cuda.empty_cache()
    dg = grape.graph_from_csr(g.off, g.col, g.w, device=local, symmetric=g.symmetric)
    g = g.to("cpu")
    torch.cuda.empty_cache()
    W = g.n * wk["walks_per_node"]
    B = min(W, args.skipgram)
    L = wk["L"]
    base, _ = weak_scaling_range(B, rank, world)
    starts = starts_per_node(g.n, wk["walks_per_node"], device=dev)[:B].contiguous()
    walks = torch.empty((B, L), dtype=torch.int32, device=dev)
    S = B * L * 2 * win
    outs = (torch.empty(S, dtype=torch.int32, device=dev), torch.empty(S, dtype=torch.int32, device=dev),
            torch.empty((S, K), dtype=torch.int32, device=dev))
    node2vec = wk["mode"] == "node2vec"
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)

    def walk(c):
        kw = dict(seed=wk["seed"], walk_id_base=base, out=walks, steps=c)
        if node2vec:
            grape.walks_node2vec(dg, starts, L, wk["p"], wk["q"], **kw)
        else:
            grape.walks_first_order(dg, starts, L, **kw)

    def pairs():
        grape.skipgram_pairs(dg, walks, win, K, seed=wk["seed"] + 1, walk_id_base=base, out=outs)

    def fused(c):   # grape_walks_skipgram: walks streamed into the pair kernel (no walk matrix)
        grape.walks_skipgram(dg, starts, L, win, K, node2vec=node2vec, p=wk["p"], q=wk["q"], seed=wk["seed"],
                             pair_seed=wk["seed"] + 1, walk_id_base=base, out=outs, steps=c)

    for _ in range(args.warmup):
        walk(None)
        pairs()
        fused(None)
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    fctr = torch.zeros(1, dtype=torch.int64, device=dev)
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        torch.cuda._sleep(int(0.1 * 1.9e9))   # GPU busy while the timed steps are enqueued (as run_ours)
        for e in evs:
            e[0].record()
            walk(ctr)
            e[1].record()
            pairs()
            e[2].record()
            fused(fctr)
            e[3].record()
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t_walk = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    t_pair = sum(e[1].elapsed_time(e[2]) for e in evs) / 1e3
    t_fused = sum(e[2].elapsed_time(e[3]) for e in evs) / 1e3
    valid = int((outs[0] != -1).sum().item())
    steps = float(ctr.item())
    tot = _allreduce(t_walk + t_pair, dist.ReduceOp.MAX, world)
    slots_all = _allreduce(float(valid * args.steps), dist.ReduceOp.SUM, world)
    peak, peak_src = _peaks()
    bytes_pair = S * (2 + K) * 4 + B * L * 4   # outputs written once + the walk matrix read once
    pair_traffic = None if (args.no_probe or rank != 0) else _dram_probe(pairs, dev)   # one more, untimed
    cpu = None
    if rank == 0 and not args.no_cpu and world == 1:
        from oracle.oracle import Oracle
        o = Oracle(*g.numpy())
        wn = walks.cpu().numpy().view(np.uint32)
        t0 = time.perf_counter()
        o.skipgram(wn[:64], win, K, seed=wk["seed"] + 1, base=base)
        per = max(time.perf_counter() - t0, 1e-4) / 64
        nrows = int(min(B, max(64, args.cpu_budget / per)))
        t0 = time.perf_counter()
        c_, _, _ = o.skipgram(wn[:nrows], win, K, seed=wk["seed"] + 1, base=base)
        dt = time.perf_counter() - t0
        cpu = {"value": float((c_ != 0xFFFFFFFF).sum()) / dt, "unit": "training pairs/s", "cores": 1,
               "kind": "oracle", "sample": f"oracle_skipgram on the first {nrows} walk rows of the batch, "
                                           f"1 thread, {dt:.1f} s (walk time not included)"}
    if rank == 0:
        line = {"metric": f"SkipGram training pairs/s (window {win}, {K} scale-free negatives each) from "
                          f"{'node2vec' if node2vec else 'first-order'} walks, walk + pair kernels",
                "value": slots_all / tot, "unit": "training pairs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32 integer",
                "data": "synthetic (seeded generator, graphgen/)",
                "config": dict(_workload_desc(k, g, wk, B), batch_walks=B, window=win, negatives=K),
                "gpu_launches": 2 * args.steps,
                "walk_steps_per_s_with_pairs": steps / (t_walk + t_pair),
                "streamed": {"path": "grape_walks_skipgram (walk rows streamed chunk by chunk through an "
                                     "L2-resident buffer into the pair kernel; no walk matrix)",
                             "ms": 1e3 * t_fused / args.steps,
                             "training_pairs_per_s": valid * args.steps / t_fused,
                             "vs_two_calls": (t_walk + t_pair) / t_fused,
                             "walk_matrix_bytes_not_materialised": B * L * 4,
                             "steps_equal": float(fctr.item()) == steps},
                "walk_steps_per_s_alone": steps / t_walk,
                "pair_kernel": {"ms": 1e3 * t_pair / args.steps, "slots": S, "valid_pairs": valid,
                                "negatives_per_s": valid * K * args.steps / t_pair},
                "roofline": {"bound": "hbm", "kernel": "skipgram_kernel (grape_skipgram_pairs)",
                             "achieved": bytes_pair * args.steps / t_pair / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": bytes_pair * args.steps / t_pair / 1e9 / peak, "traffic": pair_traffic,
                             "traffic_source": ("measured in this run: CUPTI range profiler over one untimed "
                                                "pair-kernel launch" if pair_traffic else None),
                             "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_pair,
                             "random_access": _sg_lookup_roofline(g.n, g.m, valid * K, t_pair / args.steps)},
                "cpu_baseline": cpu, "e2e": None, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dg.free()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--mode", default=None, choices=["node2vec", "first_order"],
                    help="override the config's walk mode (configs[4] names both)")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work per thread")
    ap.add_argument("--ref-budget", type=float, default=6.0)
    ap.add_argument("--traffic-per-launch", type=float, default=None,
                    help="ncu dram bytes per launch of the walk kernel (from profiles/)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--skipgram", type=int, default=0, metavar="B",
                    help="SkipGram consumer mode (§8(f) f3): B walks per step + their pairs / negatives")
    ap.add_argument("--parts", type=int, default=1,
                    help="split the tables into N parts (grape_graph_partition, §8(f) f4 layout) on this GPU")
    ap.add_argument("--window", type=int, default=5)
    ap.add_argument("--negatives", type=int, default=5)
    ap.add_argument("--no-tables", action="store_true", help="GRAPE_NO_TABLES: the v3 fenced-search walker")
    ap.add_argument("--sampler", default="rejection", choices=["rejection", "cdf", "folded"],
                    help="node2vec sampler: the default rejection rules, or the paper's CDF sampler "
                         "(grape_walks_node2vec_cdf, P:507-511)")
    ap.add_argument("--approx", type=int, default=0,
                    help="approximated walks with SUSS degree threshold d_T (grape_walks_approx; 0 = exact)")
    ap.add_argument("--layout", default="", help="force table layout fields, e.g. "
                    "record_bytes=16,guide_bytes=8,guide_factor=1,hash_h=6 (grape_table_options)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle baseline (profiling runs)")
    ap.add_argument("--no-probe", action="store_true",
                    help="do not read the walk kernel's DRAM bytes from the GPU counters (CUPTI)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the config's fixed walk list sharded by start node (north_star); "
                         "weak = the whole per-GPU workload on every rank")
    ap.add_argument("--scale-down", type=int, default=0, help="shrink the config's graph by 2^k (tests)")
    ap.add_argument("--max-walks", type=int, default=0,
                    help="walk only the first N walks of the config's list (ncu captures of the long configs)")
    ap.add_argument("--slice", default="",
                    help="R/N: walk rank R's slice of an N-rank strong-scaling run in this one process "
                         "(the per-rank launch time and its tail, measured on one GPU)")
    ap.add_argument("--device", type=int, default=None,
                    help="CUDA device of every rank (default LOCAL_RANK); tests pin two ranks to cuda:0")
    ap.add_argument("--dist-backend", default=None, choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (default nccl on GPUs)")
    ap.add_argument("--dist-tables", action="store_true",
                    help="N > 1: build the sampling tables distributed over the ranks (grape_graph_dist_*, "
                         "§8(f) f4), one part per rank; walks read every part")
    ap.add_argument("--table-budget", type=float, default=0.0,
                    help="--dist-tables: table GB per rank (default: the smallest free memory over the ranks)")
    ap.add_argument("--dump-walks", default=None, metavar="PREFIX",
                    help="save each rank's walk matrix to PREFIX.rank<r>.npy (parity tests)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.skipgram:
        run_skipgram(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
