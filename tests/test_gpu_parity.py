"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit for bit.

Walk matrices are integer work, so the bar is bit-exact equality of every
compared row plus the realised-step counter.
"""
import numpy as np
import pytest
import torch

from graphgen import CSR, config_graph, config_walks, tiny_graph, starts_per_node
from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu

PAD = 0xFFFFFFFF


@pytest.fixture(scope="module")
def grape():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2110_06196_b200 as grape
    return grape


LAYOUTS = {   # forced table layouts (grape_table_options), weighted / unweighted
    "slim": ({"guide_bytes": 8, "guide_factor": 2}, {"record_bytes": 16}),
    "compact": ({"record_bytes": 16, "guide_bytes": 8, "guide_factor": 1, "hash_h": 6},
                {"record_bytes": 8, "hash_h": 6}),
}


def _dev_graph(grape, g: CSR, symmetric=None, tables=True):
    """tables: True (automatic layout), False (GRAPE_NO_TABLES: v3 walker) or a LAYOUTS key."""
    sym = g.symmetric if symmetric is None else symmetric
    layout = LAYOUTS[tables][0 if g.w is not None else 1] if isinstance(tables, str) else None
    return grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=sym, tables=bool(tables), layout=layout)


def _run(grape, dg, starts, L, mode, p, q, seed, base=0):
    st = torch.as_tensor(np.asarray(starts, dtype=np.uint32).view(np.int32)).cuda()
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    if mode == "first_order":
        out = grape.walks_first_order(dg, st, L, seed=seed, walk_id_base=base, steps=steps)
    else:
        out = grape.walks_node2vec(dg, st, L, p, q, seed=seed, walk_id_base=base, steps=steps)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32), int(steps.item())


def _oracle(g: CSR):
    return Oracle(*g.numpy())


@pytest.mark.parametrize("tables", [True, False], ids=["v4-tables", "v3-fenced"])
def test_cfg1_every_walk_bit_exact(grape, tables):
    """configs[0]: Chung-Lu 10k nodes, first-order, 1 walk/node, L=32, seed 42 — all walks."""
    g = config_graph(1)
    wk = config_walks(1)
    starts = starts_per_node(g.n, wk["walks_per_node"]).numpy().view(np.uint32)
    dg = _dev_graph(grape, g, tables=tables)
    assert dg.info["tables"] == int(tables)
    got, steps = _run(grape, dg, starts, wk["L"], wk["mode"], 1, 1, wk["seed"])
    exp, esteps = _oracle(g).walks(starts, wk["L"], mode=wk["mode"], seed=wk["seed"])
    assert np.array_equal(got, exp)
    assert steps == esteps
    # node2vec on the same graph (unweighted, symmetric), all walks
    for p, q in [(0.5, 2.0), (1.0, 0.25), (4.0, 1.0)]:
        got, steps = _run(grape, dg, starts, 32, "node2vec", p, q, 7)
        exp, esteps = _oracle(g).walks(starts, 32, mode="node2vec", p=p, q=q, seed=7)
        assert np.array_equal(got, exp), (p, q)
        assert steps == esteps


FUZZ = [(s, n, d, directed, weighted) for s, (n, d, directed, weighted) in enumerate([
    (1, 0.0, False, False), (2, 1.0, False, True), (7, 0.4, True, False), (30, 0.15, False, True),
    (30, 0.15, True, True), (64, 0.05, True, False), (200, 0.03, False, False), (200, 0.03, False, True),
    (300, 0.02, True, True), (97, 0.3, False, True)])]


@pytest.mark.parametrize("seed,n,dens,directed,weighted", FUZZ)
@pytest.mark.parametrize("mode,p,q", [("first_order", 1, 1), ("node2vec", 0.5, 2.0), ("node2vec", 2.0, 0.5),
                                      ("node2vec", 1.0, 0.25), ("node2vec", 0.25, 4.0), ("node2vec", 4.0, 1.0),
                                      ("node2vec", 1.0, 1.0), ("node2vec", 0.3, 3.0)])
def test_fuzz_graphs_every_walk(grape, seed, n, dens, directed, weighted, mode, p, q):
    g = tiny_graph(1000 + seed, n, dens, directed=directed, weighted=weighted, self_loops=directed)
    starts = np.concatenate([np.arange(n), np.arange(n)[::-1], [n, n + 1, 2 ** 32 - 2, 2 ** 32 - 1]])
    starts = starts.astype(np.uint32)
    o = _oracle(g)
    for L in (1, 2, 3, 17, 64):
        exp, esteps = o.walks(starts, L, mode=mode, p=p, q=q, seed=seed, base=3 * seed)
        for sym, tables in ([(False, True), (True, "slim"), (False, "compact"), (False, False), (True, False)]
                            if not directed else [(False, True), (False, "slim"), (False, "compact"), (False, False)]):
            dg = _dev_graph(grape, g, symmetric=sym, tables=tables)
            got, steps = _run(grape, dg, starts, L, mode, p, q, seed, base=3 * seed)
            assert np.array_equal(got, exp), (L, sym, tables)
            assert steps == esteps


@pytest.mark.parametrize("L,base", [(3001, 2 ** 32 - 7), (70000, 11), (6, 2 ** 64 - 200), (40, 2 ** 48 + 3)])
def test_long_walks_and_wide_walk_ids(grape, L, base):
    """Rows longer than any staging unit, and walk ids whose counter word 1 is
    non-zero (crossing 2^32) or near 2^64: every walk bit-exact, default and folded
    rules, and the SkipGram slots of those rows."""
    g = tiny_graph(4242, 60, 0.08, weighted=True)
    o = _oracle(g)
    starts = np.concatenate([np.arange(g.n), [g.n + 5]]).astype(np.uint32)[: (3 if L > 10000 else 200)]
    dg = _dev_graph(grape, g)
    for mode, p, q in (("node2vec", 0.5, 2.0), ("first_order", 1, 1)):
        exp, esteps = o.walks(starts, L, mode=mode, p=p, q=q, seed=5, base=base)
        got, steps = _run(grape, dg, starts, L, mode, p, q, 5, base=base)
        assert np.array_equal(got, exp) and steps == esteps, mode
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    fo = grape.walks_node2vec_folded(dg, st, L, 0.25, 4.0, seed=5, walk_id_base=base)
    efo, _ = o.walks_folded(starts, L, p=0.25, q=4.0, seed=5, base=base)
    assert np.array_equal(fo.cpu().numpy().view(np.uint32), efo)
    if L * len(starts) <= 200 * 3001 and base < 2 ** 63:
        c, x, ng = grape.skipgram_pairs(dg, fo[:2], 3, 2, seed=1, walk_id_base=base)
        ec, ex, eng = o.skipgram(efo[:2], 3, 2, seed=1, base=base)
        assert np.array_equal(c.cpu().numpy().view(np.uint32), ec)
        assert np.array_equal(ng.cpu().numpy().view(np.uint32), eng)


def test_u64_prefix_path(grape):
    """Row sums >= 2^32 force the u64 prefix layout; results stay bit-exact."""
    g = tiny_graph(5, 40, 0.5, weighted=True)
    rng = np.random.default_rng(0)
    w = rng.integers(2 ** 30, 2 ** 32 - 1, g.m, dtype=np.uint64).astype(np.uint32)
    # keep it symmetric-weighted is not required for correctness
    g.w = torch.from_numpy(w.view(np.int32))
    dg = _dev_graph(grape, g)
    assert dg.info["cw_bytes"] == 8
    assert dg.info["tables"] == 0   # outside the tables' u32 prefix range: v3 walker
    starts = np.arange(g.n, dtype=np.uint32)
    for mode, p, q in [("first_order", 1, 1), ("node2vec", 0.5, 2.0), ("node2vec", 1.0, 0.25)]:
        got, steps = _run(grape, dg, starts, 50, mode, p, q, 11)
        exp, esteps = _oracle(g).walks(starts, 50, mode=mode, p=p, q=q, seed=11)
        assert np.array_equal(got, exp)
        assert steps == esteps


def test_edge_cases(grape):
    g = tiny_graph(9, 20, 0.1, directed=True, weighted=True)
    dg = _dev_graph(grape, g)
    # num_walks = 0
    out = grape.walks_node2vec(dg, torch.empty(0, dtype=torch.int32, device="cuda"), 5, 0.5, 2.0)
    assert out.shape == (0, 5)
    # all starts invalid -> all PAD
    got, steps = _run(grape, dg, [20, 21, 2 ** 32 - 1], 7, "node2vec", 0.5, 2.0, 1)
    assert np.all(got == PAD) and steps == 0
    # a graph with no arcs: every row is [start, PAD, ...]
    e = CSR(5, torch.zeros(6, dtype=torch.int64), torch.zeros(0, dtype=torch.int32), None, True)
    de = _dev_graph(grape, e)
    got, steps = _run(grape, de, np.arange(5), 4, "node2vec", 2.0, 0.5, 1)
    assert np.all(got[:, 0] == np.arange(5)) and np.all(got[:, 1:] == PAD) and steps == 0


def test_host_buffer_path_equals_device_path(grape):
    g = config_graph(2, scale_down=6)
    dg = _dev_graph(grape, g)
    starts = starts_per_node(g.n, 3)
    dev = grape.walks_node2vec(dg, starts.cuda(), 40, 0.5, 2.0, seed=42, walk_id_base=17)
    steps = torch.zeros(1, dtype=torch.int64)
    host = grape.walks_node2vec(dg, starts, 40, 0.5, 2.0, seed=42, walk_id_base=17, steps=steps)
    assert not host.is_cuda
    assert torch.equal(dev.cpu(), host)
    dsteps = torch.zeros(1, dtype=torch.int64, device="cuda")
    grape.walks_node2vec(dg, starts.cuda(), 40, 0.5, 2.0, seed=42, walk_id_base=17, steps=dsteps)
    assert int(dsteps.item()) == int(steps.item())


@pytest.mark.parametrize("chunk_mb", ["1", "3"])
def test_host_buffer_path_many_chunks(grape, monkeypatch, chunk_mb):
    """The staged pipeline with many chunks (and a ragged last one), the staging buffer
    cached in the graph reused across calls of different sizes."""
    monkeypatch.setenv("GRAPE_HOST_CHUNK_MB", chunk_mb)
    g = config_graph(2, scale_down=6)
    dg = _dev_graph(grape, g)
    for W, L in ((g.n * 4 + 7, 40), (g.n + 3, 113), (5, 3)):
        starts = starts_per_node(g.n, 5)[:W]
        assert starts.numel() * L * 4 > 2 * (int(chunk_mb) << 20) or W == 5
        dev = grape.walks_node2vec(dg, starts.cuda(), L, 0.5, 2.0, seed=9, walk_id_base=3)
        steps = torch.zeros(1, dtype=torch.int64)
        host = grape.walks_node2vec(dg, starts, L, 0.5, 2.0, seed=9, walk_id_base=3, steps=steps)
        assert torch.equal(dev.cpu(), host), (W, L)
        dsteps = torch.zeros(1, dtype=torch.int64, device="cuda")
        grape.walks_node2vec(dg, starts.cuda(), L, 0.5, 2.0, seed=9, walk_id_base=3, steps=dsteps)
        assert int(dsteps.item()) == int(steps.item())


def test_sharding_and_determinism(grape):
    """Rank slices [r W/G, (r+1) W/G) with walk_id_base = slice start reproduce the
    single call bit for bit; re-running is deterministic."""
    g = config_graph(2, scale_down=5)
    dg = _dev_graph(grape, g)
    starts = starts_per_node(g.n, 2).cuda()
    W = starts.numel()
    full = grape.walks_node2vec(dg, starts, 30, 0.5, 2.0, seed=42)
    again = grape.walks_node2vec(dg, starts, 30, 0.5, 2.0, seed=42)
    assert torch.equal(full, again)
    for G in (2, 3, 8):
        parts = []
        for r in range(G):
            lo, hi = r * W // G, (r + 1) * W // G
            parts.append(grape.walks_node2vec(dg, starts[lo:hi], 30, 0.5, 2.0, seed=42, walk_id_base=lo))
        assert torch.equal(torch.cat(parts), full)


def test_specialisation_identities(grape):
    g = config_graph(1)
    dg = _dev_graph(grape, g)
    dn = _dev_graph(grape, g, symmetric=False)
    ones = CSR(g.n, g.off, g.col, torch.ones(g.m, dtype=torch.int32), True)
    dw = _dev_graph(grape, ones)
    dv3 = _dev_graph(grape, g, tables=False)
    starts = starts_per_node(g.n, 1).cuda()
    a = grape.walks_node2vec(dg, starts, 32, 1.0, 1.0, seed=3)
    b = grape.walks_first_order(dg, starts, 32, seed=3)
    assert torch.equal(a, b)
    for p, q in [(0.5, 2.0), (1.0, 0.25), (2.0, 1.0)]:
        x = grape.walks_node2vec(dg, starts, 32, p, q, seed=3)
        y = grape.walks_node2vec(dn, starts, 32, p, q, seed=3)   # no symmetric trick
        z = grape.walks_node2vec(dw, starts, 32, p, q, seed=3)   # weighted, all ones
        v = grape.walks_node2vec(dv3, starts, 32, p, q, seed=3)  # fenced-search walker
        assert torch.equal(x, y) and torch.equal(x, z) and torch.equal(x, v)


FULL = [(2, "node2vec"), (3, "node2vec"), (4, "node2vec"), (5, "node2vec"), (5, "first_order"),
        (6, "node2vec"),   # 6: beyond BASELINE, 2.2e9 arcs (> 2^31: the lifted index range)
        (7, "node2vec")]   # 7: beyond BASELINE, 4.8e9 arcs (> 2^32: the wide walker), first 2e7 walks


@pytest.mark.parametrize("k,mode", FULL, ids=[f"cfg{k}-{m}" for k, m in FULL])
def test_full_size_config_sampled(grape, k, mode):
    """BASELINE configs at full size, in bench.py's launch configuration (one call
    over all walks of the config): a seeded sample of GPU rows — 10^4 random wids,
    every walk starting at one of the 100 highest-degree nodes, and every walk
    starting at one of 100 sinks (out-degree 0; directed configs) — each compared
    with the oracle's walk recomputed alone (the counter-based RNG makes walk i a
    function of (seed, wid) alone); plus the step counter against the matrix and
    invariants on the whole matrix."""
    wk = config_walks(k)
    g = config_graph(k, device="cuda")
    torch.cuda.empty_cache()
    if k in (6, 7):   # past the automatic layout's 68 GB gather-reach cap: give the tables 100 GB
        dg = grape.graph_from_csr(g.off, g.col, g.w, device=0, symmetric=g.symmetric,
                                  layout={"table_budget_bytes": int(100e9)})
        assert g.m > 2 ** 31 and dg.info["tables"] == 1   # the table walker, past the old 2^31-arc range
        assert dg.info["wide"] == int(k == 7) and (k == 6 or g.m > 2 ** 32)
    else:
        dg = _dev_graph(grape, g)
    deg = (g.off[1:] - g.off[:-1])
    hubs = torch.topk(deg, 100).indices.cpu().numpy()
    sink_all = torch.nonzero(deg == 0).flatten()
    n_sinks = sink_all.numel()
    pick = torch.randperm(n_sinks, generator=torch.Generator().manual_seed(k))[:100]
    sinks = sink_all[pick.to(sink_all.device)].cpu().numpy()
    del sink_all
    del deg
    gc = g.to("cpu")   # the library holds its own copy: room for the walk matrix
    del g
    torch.cuda.empty_cache()
    starts = starts_per_node(gc.n, wk["walks_per_node"], device="cuda")
    if k == 7:   # the first 2e7 walks of the list (an 8 GB walk matrix next to 67 GB of tables)
        starts = starts[:20_000_000].contiguous()
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    if mode == "node2vec":
        out = grape.walks_node2vec(dg, starts, wk["L"], wk["p"], wk["q"], seed=wk["seed"], steps=steps)
    else:
        out = grape.walks_first_order(dg, starts, wk["L"], seed=wk["seed"], steps=steps)
    torch.cuda.synchronize()
    W = starts.numel()
    # whole-matrix checks on the device, in row chunks: rows start at their start
    # node, PAD only as a suffix, realised steps = non-PAD entries - 1 per row
    assert torch.equal(out[:, 0], starts)
    realised = 0
    for lo in range(0, W, 1 << 23):
        pad = out[lo:lo + (1 << 23)] == -1
        assert not bool((pad[:, :-1] & ~pad[:, 1:]).any())
        realised += int((~pad).sum(dim=1, dtype=torch.int32).sum().item()) - pad.shape[0]
    del pad
    assert realised == int(steps.item())
    rng = np.random.default_rng(k)
    if W < gc.n * wk["walks_per_node"]:   # (k = 7) a prefix of the walk list: the hubs / sinks inside it
        hubs, sinks = hubs[hubs < W], sinks[sinks < W]
        n_sinks = min(n_sinks, len(sinks))
    # every walk whose start is a hub or a sink: wid = it * n + node for every iteration it
    special = np.concatenate([hubs, sinks]).astype(np.int64)
    its = np.arange(wk["walks_per_node"], dtype=np.int64) * gc.n
    sample = np.concatenate([rng.integers(0, W, 10_000), (special[None, :] + its[:, None]).ravel(), [0, W - 1]])
    sample = np.unique(sample)
    assert len(sample) >= 10_000
    idx = torch.as_tensor(sample, device="cuda")
    host_out = out[idx].cpu().numpy().view(np.uint32)
    st_np = starts[idx].cpu().numpy().view(np.uint32)
    del out
    dg.free()
    torch.cuda.empty_cache()
    o = _oracle(gc)
    for r, i in enumerate(sample):
        exp, _ = o.walks(st_np[r:r + 1], wk["L"], mode=mode, p=wk["p"], q=wk["q"], seed=wk["seed"], base=int(i))
        assert np.array_equal(host_out[r], exp[0]), int(i)
    # the GPU rows of walks from sinks (directed configs): [start, PAD, ...]
    if len(sinks):
        assert len(sinks) == min(100, n_sinks)   # cfg3: isolated nodes; cfg4: a few; cfg5: the 5% sinks
        at = {int(i): r for r, i in enumerate(sample)}
        for it in range(wk["walks_per_node"]):
            for s_ in sinks:
                row = host_out[at[int(s_) + it * gc.n]]
                assert row[0] == s_ and np.all(row[1:] == PAD), int(s_)
    # and the GPU rows from hubs were all compared above
    for h in hubs:
        assert int(h) in {int(i) for i in sample}


def test_invalid_inputs_rejected(grape):
    good = tiny_graph(3, 10, 0.3)
    off, col = good.off.clone(), good.col.clone()
    with pytest.raises(grape.GrapeError) as ei:
        grape.graph_from_csr(off, col.flip(0))            # unsorted rows
    assert ei.value.status == grape.GRAPE_EINVAL
    bad = col.clone(); bad[0] = 10
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(off, bad)                     # col >= n
    bad_off = off.clone(); bad_off[-1] += 1
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(bad_off, col)                 # off[n] != m
    w = torch.ones(good.m, dtype=torch.int32); w[3] = 0
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(off, col, w)                  # weight 0
    d = tiny_graph(4, 10, 0.3, directed=True)
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(d.off, d.col, symmetric=True)   # asymmetric with SYMMETRIC (caught by the table build)
    with pytest.raises(grape.GrapeError):
        grape.graph_from_csr(d.off, d.col, symmetric=True, tables=False)   # (by the validation pass)
    with pytest.raises(grape.GrapeError):   # tables that do not fit: the v3 walker, checked after the attempt
        grape.graph_from_csr(d.off, d.col, symmetric=True, layout={"table_budget_bytes": 1})
    dg = grape.graph_from_csr(off, col, symmetric=True)
    st = torch.arange(10, dtype=torch.int32, device="cuda")
    for p, q in [(0.0, 1.0), (1.0, -2.0), (float("nan"), 1.0), (2.0 ** 25, 1.0)]:
        with pytest.raises(grape.GrapeError):
            grape.walks_node2vec(dg, st, 5, p, q)
    with pytest.raises(grape.GrapeError):
        grape.walks_node2vec(dg, st, 0, 1.0, 1.0)
    with pytest.raises(ValueError):         # host starts with a device out (the binding refuses it)
        grape.walks_node2vec(dg, st.cpu(), 5, 1.0, 1.0, out=torch.empty(10, 5, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("tables", [True, "slim", "compact", False], ids=["v4-tables", "v4-slim", "v4-compact",
                                                                         "v3-fenced"])
@pytest.mark.parametrize("mode,p,q,sym,weighted", [("node2vec", 0.5, 2.0, True, True), ("node2vec", 1.0, 0.25, False, False),
                                                   ("first_order", 1, 1, True, True), ("node2vec", 2.0, 1.0, True, False),
                                                   ("node2vec", 0.25, 4.0, False, True)])
def test_stats_build_matches_and_counts(grape, mode, p, q, sym, weighted, tables):
    """grape_walks_stats: the counting build writes the same walks; its attempt and
    step counters equal the oracle's (attempts = draws of node2vec steps s >= 2
    plus one draw per first-order / first step)."""
    g = tiny_graph(31, 300, 0.03, directed=not sym, weighted=weighted)
    dg = _dev_graph(grape, g, tables=tables)
    starts = np.concatenate([np.arange(g.n), [g.n + 3]]).astype(np.uint32)
    st = torch.as_tensor(starts.view(np.int32)).cuda()
    plain = grape.walks_node2vec(dg, st, 40, p, q, seed=5) if mode == "node2vec" else \
        grape.walks_first_order(dg, st, 40, seed=5)
    out, stats = grape.walks_stats(dg, st, 40, node2vec=mode == "node2vec", p=p, q=q, seed=5)
    torch.cuda.synchronize()
    assert torch.equal(out, plain)
    exp, esteps, eatt = _oracle(g).walks(starts, 40, mode=mode, p=p, q=q, seed=5, with_attempts=True)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), exp)
    assert stats["steps"] == esteps
    if mode == "node2vec" and not (p == 1 and q == 1):
        first = int(np.sum(exp[:, 1] != PAD))   # walks that made their (first-order) first step
        assert stats["attempts"] == eatt + first
    else:
        assert stats["attempts"] == esteps
    assert stats["start_loads"] == len(starts)
    kinds = ("node_loads", "xnode_loads", "cw_probes", "col_probes", "col_loads", "start_loads",
             "guide_loads", "hash_probes")
    assert stats["sector_loads"] == sum(stats[k] for k in kinds)
    if tables is False:
        assert stats["col_loads"] == stats["attempts"]
        assert stats["guide_loads"] == stats["hash_probes"] == stats["alu_decisions"] == 0
        if not weighted:
            assert stats["cw_probes"] == 0
    else:
        # v4: an attempt is decided from registers or reads its proposal: weighted,
        # one guide entry (rows of degree > 1) and the record when it is needed;
        # unweighted, the record; an accepted proposal whose membership test ran
        # after the read re-reads its record.  Node records are read for starts only.
        assert stats["xnode_loads"] == stats["cw_probes"] == stats["col_probes"] == 0
        proposals = stats["attempts"] - stats["alu_decisions"]
        assert 0 <= stats["alu_decisions"] <= stats["attempts"]
        if weighted:   # (fat guide: an accepted proposal re-reads its guide entry after a membership test)
            assert stats["guide_loads"] <= proposals + stats["membership_tests"]
        else:
            assert stats["guide_loads"] == 0
            assert proposals <= stats["col_loads"] <= proposals + stats["membership_tests"]
        assert stats["hash_probes"] >= stats["membership_tests"]
        if tables != "compact":
            assert stats["node_loads"] <= len(starts)
        else:
            assert stats["node_loads"] <= len(starts) + esteps
        if mode == "node2vec" and p < min(1.0, q):
            assert stats["alu_decisions"] > 0
