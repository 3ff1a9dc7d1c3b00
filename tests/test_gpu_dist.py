"""Partitioned D-iteration on emulated ranks: G host threads share one GPU
through a LocalGroup (the collectives become host barriers + device copies; no kernel waits for
another rank). Every kernel of the multi-GPU sweep runs: select on the owned range, the push
that routes remote targets into R with first-touch lists, pack, the exchange, apply, and the
finaliser on the allreduced sums. The NCCL backend differs only in how the bytes move."""
import numpy as np
import pytest

import digen
import oracle
from conftest import load_pins
from gpu_util import l1, need_gpu
from oracle import definition as defn

pytestmark = pytest.mark.gpu
D = 0.85
torch = pytest.importorskip("torch")


def run(src, dst, n, G, solves, reorder=True, B=None, **kw):
    """Build the partitioned graph on G emulated ranks and run `solves` (list of solve kwargs);
    returns per solve: (assembled H, assembled F, stats of rank 0, all ranks' stats, ranges)."""
    import paper_1204_6255_b200 as di
    from paper_1204_6255_b200.dist import assemble, run_local_group

    def fn(r, grp):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            g = di.Graph(src, dst, n, rank=r, world=G, group=grp, stream=stream, reorder=reorder, **kw)
            out = []
            for sk in solves:
                sk = dict(sk)
                if B is not None:
                    sk["B"] = B[g.lo:g.hi]
                st = g.solve(**sk)
                H = g.history().cpu().numpy()
                l1f, F = g.residual(return_F=True)
                out.append((H, F.cpu().numpy(), st, l1f))
            rng = (g.lo, g.hi)
            g.free()
        return rng, out

    res = run_local_group(G, fn)
    ranges = [r for r, _ in res]
    outs = []
    for k in range(len(solves)):
        H = assemble([o[k][0] for _, o in res], ranges, n)
        F = assemble([o[k][1] for _, o in res], ranges, n)
        sts = [o[k][2] for _, o in res]
        l1s = [o[k][3] for _, o in res]
        assert len(set(l1s)) == 1            # di_residual is collective: same value everywhere
        outs.append((H, F, sts[0], sts, ranges))
    return outs


def same_stats(sts):
    keys = ("sweeps", "selected_total", "link_diffusions", "starvation_fallbacks", "residual_l1",
            "dangling_absorbed", "converged")
    for k in keys:
        assert len({s[k] for s in sts}) == 1, (k, [s[k] for s in sts])


@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("asynchronous", [False, True])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_pins_partitioned(G, asynchronous, p2p):
    """T1 on partitions: the exact rationals of tests/golden/pins.txt (graphs with >= G nodes),
    bulk sweeps and asynchronous cycles (R7 on every rank, one exchange per cycle); the lists
    through peer memory (fused compaction + transfer) or through the backend's send/recv."""
    need_gpu()
    for name, n, links, X in load_pins():
        if n < G:
            continue
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        for variant in ("sop", "cyc"):
            H, F, st, sts, _ = run(src, dst, n, G, [dict(d=D, tol=1e-16, variant=variant,
                                                         asynchronous=asynchronous, p2p=p2p)])[0]
            same_stats(sts)
            assert st["converged"] == 1, (name, st)
            assert all(s_["p2p_exchanges"] == (s_["sweeps"] - s_["dense_exchanges"] if p2p else 0)
                       for s_ in sts)
            assert l1(H, [float(x) for x in X]) <= 1e-14, (name, variant, H)


@pytest.mark.parametrize("asynchronous", [False, True])
@pytest.mark.parametrize("G", [2, 4])
def test_random_vs_dense_partitioned(G, asynchronous):
    """T2 on partitions: random graphs with self-loops, duplicates, dangling nodes."""
    need_gpu()
    for seed in range(25):
        src, dst, n = digen.small_random(seed)
        if n < G:
            continue
        X = defn.solve_dense(src, dst, n, D)
        kw = dict(d=D, tol=1e-15, asynchronous=asynchronous)
        for H, F, st, sts, ranges in run(src, dst, n, G, [dict(variant="sop", **kw),
                                                           dict(variant="cyc", **kw)]):
            same_stats(sts)
            assert st["converged"] == 1
            assert l1(H, X) <= 1e-13, (seed, G)


@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("asynchronous", [False, True])
@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("variant", ["sop", "cyc"])
def test_north_star_parity_partitioned(G, variant, asynchronous, p2p):
    """T11 / T10 on partitions: C1 at tol 1e-10 vs the oracle (1e-9, and the G19 bound against
    the tight 1e-13 oracle run); the partition and the exchange counters are sane."""
    need_gpu()
    src, dst, n = digen.make("c1", seed=1)
    (H, F, st, sts, ranges), = run(src, dst, n, G, [dict(d=D, tol=1e-10, variant=variant,
                                                         asynchronous=asynchronous,
                                                         exchange="sparse", p2p=p2p)])
    same_stats(sts)
    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant=variant)
    assert l1(H, Ho) <= 1e-9
    Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant=variant)
    assert l1(H, Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D)
    # partition: contiguous, non-empty, balanced on 20 B/link + 12 B/node
    out = np.bincount(src, minlength=n).astype(np.int64)
    w = 20 * out + 12
    W = w.sum()
    for lo, hi in ranges:
        assert hi > lo
        assert w[lo:hi].sum() <= W / G + w.max() + 12
    # the exchange moved something, and never more than one entry per (remote node, sweep)
    assert all(s["exchange_entries"] > 0 for s in sts)
    for s, (lo, hi) in zip(sts, ranges):
        assert s["exchange_entries"] <= (n - (hi - lo)) * s["sweeps"]
        assert s["exchange_bytes"] == 12 * s["exchange_entries"] + 16 * s["exchange_cold"]
        assert s["p2p_exchanges"] == (s["sweeps"] if p2p else 0)


@pytest.mark.parametrize("asynchronous", [False, True])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_dense_exchange_partitioned(G, asynchronous):
    """The dense fallback of the exchange (a per-owner reduction of the
    remote accumulator): exact pins, C1 at the north_star gate, F = B + P.H - H mid-solve, its
    byte count (8 B per remote node per sweep); and the automatic choice, which must take it on
    a graph whose every sweep touches every remote node, and still reach the same fixed point."""
    need_gpu()
    for name, n, links, X in load_pins():
        if n < G:
            continue
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        H, F, st, sts, _ = run(src, dst, n, G, [dict(d=D, tol=1e-16, asynchronous=asynchronous,
                                                     exchange="dense")])[0]
        same_stats(sts)
        assert st["converged"] == 1 and l1(H, [float(x) for x in X]) <= 1e-14, name
    src, dst, n = digen.make("c1", seed=1)
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    kw = dict(d=D, variant="sop", asynchronous=asynchronous)
    res = run(src, dst, n, G, [dict(tol=1e-10, exchange="dense", **kw),
                               dict(tol=1e-300, max_sweeps=3, exchange="dense", **kw),
                               dict(tol=1e-10, exchange="auto", **kw)])
    for H, F, st, sts, ranges in (res[0], res[2]):
        same_stats(sts)
        assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
        assert l1(H, Ho) <= 1e-9
    H, F, st, sts, ranges = res[0]
    for s_, (lo, hi) in zip(sts, ranges):
        assert s_["dense_exchanges"] == s_["sweeps"] and s_["exchange_entries"] == 0
        assert s_["exchange_bytes"] == 8 * (n - (hi - lo)) * s_["sweeps"]
    H, F, st, sts, ranges = res[1]
    assert st["sweeps"] == 3 and np.all(F >= 0)
    assert np.abs(F - (B + P @ H - H)).max() <= 1e-15
    # 40 random out-links per node: every bulk DI-CYC sweep touches ~every remote node, so the
    # lists (12 B per entry) outweigh the reduction (8 B per remote node) and auto goes dense,
    # with a sparse sweep every 5th to measure again
    rng = np.random.default_rng(G)
    n = 3000
    s2 = np.repeat(np.arange(n, dtype=np.int32), 40)
    t2 = rng.integers(0, n, 40 * n).astype(np.int32)
    X, _, _ = oracle.di(s2, t2, n, d=D, tol=1e-15, variant="cyc")
    H, F, st, sts, _ = run(s2, t2, n, G, [dict(d=D, tol=1e-13, variant="cyc", exchange="auto",
                                               asynchronous=asynchronous)])[0]
    same_stats(sts)
    assert len({s_["dense_exchanges"] for s_ in sts}) == 1     # every rank takes the same choice
    assert st["converged"] == 1 and l1(H, X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
    if not asynchronous:
        assert 0 < st["dense_exchanges"] < st["sweeps"]


@pytest.mark.parametrize("G", [2, 3, 4])
def test_dist_async(G):
    """F2 (DI_DIST_ASYNC): asynchronous cycles on every rank with no collective between two
    cycles; remote fluid through the peer-memory rings; meetings every 4 cycles. Exact pins, random
    graphs vs the dense solve, C1 at the north_star gate (vs the oracle, both to 1e-10), the
    invariant F = B + P.H - H and conservation at a max_sweeps stop (the meeting drains every
    ring), global counters identical on every rank."""
    need_gpu()
    kw = dict(d=D, asynchronous=True, dist_async=True)
    for name, n, links, X in load_pins():
        if n < G:
            continue
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        for variant in ("sop", "cyc"):
            H, F, st, sts, _ = run(src, dst, n, G, [dict(tol=1e-16, variant=variant, **kw)])[0]
            same_stats(sts)
            assert st["converged"] == 1 and st["meetings"] >= 1, (name, st)
            assert l1(H, [float(x) for x in X]) <= 1e-14, (name, variant, H)
    for seed in range(0, 25, 3):
        src, dst, n = digen.small_random(seed)
        if n < G:
            continue
        X = defn.solve_dense(src, dst, n, D)
        H, F, st, sts, _ = run(src, dst, n, G, [dict(tol=1e-15, variant="sop", **kw)])[0]
        same_stats(sts)
        assert st["converged"] == 1 and l1(H, X) <= 1e-13, seed
    src, dst, n = digen.make("c1", seed=1)
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    outd = np.bincount(src, minlength=n)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    res = run(src, dst, n, G, [dict(tol=1e-10, variant="sop", **kw),
                               dict(tol=1e-300, variant="sop", max_sweeps=6, **kw),
                               dict(tol=1e-10, variant="sop", profile=True, **kw)])
    assert res[2][2]["push_launches"] == res[2][2]["sweeps"] and res[2][2]["push_ms"] > 0
    H, F, st, sts, _ = res[0]
    same_stats(sts)
    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
    assert abs(F.sum() - st["residual_l1"]) <= 1e-18
    assert l1(H, Ho) <= 1e-9
    assert st["meetings"] == -(-st["sweeps"] // 4) + 1
    for s_ in sts:   # lists moved through the rings, at most one entry per (remote node, cycle)
        assert 0 < s_["exchange_entries"] <= n * s_["sweeps"]
        assert s_["exchange_bytes"] == 12 * s_["exchange_entries"] + 16 * s_["exchange_cold"]
    H, F, st, sts, _ = res[1]
    assert st["sweeps"] == 6 and st["converged"] == 0 and np.all(F >= 0)
    assert np.abs(F - (B + P @ H - H)).max() <= 1e-15
    cons = F.sum() + (1 - D) * H[outd > 0].sum() + H[outd == 0].sum()
    assert abs(cons - (1 - D)) <= 1e-14


@pytest.mark.parametrize("G", [2, 3])
def test_local_links(G):
    """DI_LOCAL_LINKS: every rank passes only the links of its own sources, for node ranges the
    caller chose (equal node counts here, not the library's balanced ranges); in-degrees are
    summed across ranks. C1 to the north_star gate (synchronous cycles, F2), a random graph with
    loops and duplicates vs the dense solve; a link outside the range or ranges that do not tile
    [0, n) fail on every rank."""
    need_gpu()
    import paper_1204_6255_b200 as di
    from paper_1204_6255_b200.dist import assemble, run_local_group

    def solve_local(src, dst, n, solves, cut=None):
        bounds = [n * r // G for r in range(G + 1)] if cut is None else cut

        def fn(r, grp):
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                lo, hi = bounds[r], bounds[r + 1]
                m = (src >= lo) & (src < hi)
                g = di.Graph(src[m], dst[m], n, rank=r, world=G, group=grp, stream=stream,
                             local_range=(lo, hi))
                assert g.range() == (lo, hi)
                out = []
                for sk in solves:
                    st = g.solve(**sk)
                    out.append((g.history().cpu().numpy(), st))
                g.free()
            return (lo, hi), out

        res = run_local_group(G, fn)
        return [(assemble([o[k][0] for _, o in res], [rg for rg, _ in res], n), [o[k][1] for _, o in res])
                for k in range(len(solves))]

    src, dst, n = digen.make("c1", seed=1)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    for H, sts in solve_local(src, dst, n, [dict(d=D, tol=1e-10, asynchronous=True),
                                            dict(d=D, tol=1e-10, asynchronous=True, dist_async=True),
                                            dict(d=D, tol=1e-10)]):
        same_stats(sts)
        assert sts[0]["converged"] == 1 and l1(H, Ho) <= 1e-9
        assert sts[0]["equivalent_iterations"] == sts[0]["link_diffusions"] / len(src)
    s2, t2, n2 = digen.small_random(5, n_max=300)
    X = defn.solve_dense(s2, t2, n2, D) if n2 <= 64 else oracle.di(s2, t2, n2, d=D, tol=1e-15)[0]
    (H, sts), = solve_local(s2, t2, n2, [dict(d=D, tol=1e-15, asynchronous=True)])
    assert sts[0]["converged"] == 1 and l1(H, X) <= 1e-13 * max(1, n2 / 64)

    def bad_link(r, grp):   # rank 0 passes one link of rank 1's range: every rank fails
        lo, hi = [0, n // 2, n][r], [n // 2, n, n][r]
        m = (src >= lo) & (src < hi)
        s_, t_ = src[m], dst[m]
        if r == 0:
            s_ = np.concatenate([s_, np.array([n - 1], np.int32)])
            t_ = np.concatenate([t_, np.array([0], np.int32)])
        with pytest.raises(di.DIError) as ei:
            di.Graph(s_, t_, n, rank=r, world=2, group=grp, local_range=(lo, hi))
        assert ei.value.status == di.DI_EINVAL
        return str(ei.value)

    msgs = run_local_group(2, bad_link)
    assert "outside this rank's range" in msgs[0] and "another rank" in msgs[1]

    def gap(r, grp):        # ranges [0, n/2) and [n/2 + 1, n): not a tiling
        lo, hi = [(0, n // 2), (n // 2 + 1, n)][r]
        m = (src >= lo) & (src < hi)
        with pytest.raises(di.DIError) as ei:
            di.Graph(src[m], dst[m], n, rank=r, world=2, group=grp, local_range=(lo, hi))
        assert ei.value.status == di.DI_EINVAL and "tile" in str(ei.value)

    run_local_group(2, gap)

    def empty_range(r, grp):   # rank 1 passes an empty range: both ranks fail, neither hangs
        lo, hi = [(0, n), (n, n)][r]
        m = (src >= lo) & (src < hi)
        with pytest.raises(di.DIError) as ei:
            di.Graph(src[m], dst[m], n, rank=r, world=2, group=grp, local_range=(lo, hi))
        assert ei.value.status == di.DI_EINVAL
        return str(ei.value)

    msgs = run_local_group(2, empty_range)
    assert "another rank" in msgs[0] and "0 <= dist->lo < dist->hi" in msgs[1]


def test_cyc_neumann_partitioned():
    """T7 on partitions: bulk DI-CYC without loops is the Neumann series, F_n = P^n B and
    H_n = sum_{k<n} P^k B, whatever the partition (the exchange only moves where fluid is added)."""
    need_gpu()
    src, dst, n = digen.make("c1")
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    solves = [dict(d=D, tol=1e-300, variant="cyc", max_sweeps=k) for k in range(1, 9)]
    res = run(src, dst, n, 3, solves)
    Fn, Hn = B.copy(), np.zeros(n)
    for k, (H, F, st, sts, _) in enumerate(res, start=1):
        Hn = Hn + Fn
        Fn = P @ Fn
        assert st["sweeps"] == k
        nz = Fn > 0
        assert np.array_equal(F > 0, nz)
        assert np.max(np.abs(F[nz] - Fn[nz]) / Fn[nz]) <= 1e-13
        assert np.max(np.abs(H - Hn) / np.maximum(Hn, 1e-300)) <= 1e-13


def test_invariants_and_matches_single_gpu():
    """T8 mid-solve on partitions (F = B + P.H - H, conservation) and T11's 'same sweep count
    within 1' against the single-GPU solve, on C1 and a host-block graph; custom B; resume."""
    need_gpu()
    from gpu_util import upload
    src, dst, n = digen.make("c1", seed=2)
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    outd = np.bincount(src, minlength=n)
    for H, F, st, sts, _ in run(src, dst, n, 4, [dict(d=D, tol=1e-300, variant="sop", max_sweeps=k)
                                                 for k in (1, 4, 9)]):
        assert np.all(F >= 0)
        assert np.abs(F - (B + P @ H - H)).max() <= 1e-15
        cons = F.sum() + (1 - D) * H[outd > 0].sum() + H[outd == 0].sum()
        assert abs(cons - (1 - D)) <= 1e-14
    g = upload(src, dst, n)
    st1 = g.solve(d=D, tol=1e-10, variant="sop")
    H1 = g.history().cpu().numpy()
    g.free()
    H, F, st, sts, _ = run(src, dst, n, 4, [dict(d=D, tol=1e-10, variant="sop")])[0]
    assert abs(st["sweeps"] - st1["sweeps"]) <= 1
    assert l1(H, H1) <= 2e-10 / (1 - D)
    # custom B (each rank passes its slice in the caller's numbering) + resume
    rng = np.random.default_rng(3)
    Bc = rng.random(n) * (1 - D) / n * 2
    X = defn.solve_sparse(src, dst, n, D, B=Bc)
    res = run(src, dst, n, 3, [dict(d=D, tol=1e-12, variant="sop", max_sweeps=6),
                               dict(d=D, tol=1e-12, variant="sop", resume=True)], B=Bc)
    assert res[0][2]["converged"] == 0 and res[0][2]["sweeps"] == 6
    assert res[1][2]["converged"] == 1
    assert l1(res[1][0], X) <= 1e-12 / (1 - D)


def test_edge_cases_partitioned():
    """n == G (one node per rank), no links at all, hubs above the chunk size, no relabelling,
    self-loops kept, dedup; and C2 (10^6 nodes) at G = 2 vs the oracle."""
    need_gpu()
    # one node per rank: 0 -> 1 -> 2 -> 3 -> 0 ring plus a self-loop
    src = np.array([0, 1, 2, 3, 2], np.int32)
    dst = np.array([1, 2, 3, 0, 2], np.int32)
    X = defn.solve_dense(src, dst, 4, D)
    H, *_ = run(src, dst, 4, 4, [dict(d=D, tol=1e-15)])[0]
    assert l1(H, X) <= 1e-14
    # no links: every node dangling, X = (1-d)/N
    H, F, st, _, _ = run(np.zeros(0, np.int32), np.zeros(0, np.int32), 1000, 3, [dict(d=D, tol=1e-12)])[0]
    assert st["sweeps"] == 1 and np.allclose(H, (1 - D) / 1000, rtol=0, atol=1e-18)
    # hubs (push bin C) crossing the partition, duplicates, no relabelling
    n = 20000
    rng = np.random.default_rng(7)
    s = rng.integers(0, n, 4 * n).astype(np.int32)
    t = rng.integers(0, n, 4 * n).astype(np.int32)
    s = np.concatenate([s, np.zeros(15000, np.int32), s[:100]])
    t = np.concatenate([t, np.arange(1, 15001, dtype=np.int32), t[:100]])
    # reference: the (pinned) sequential oracle run tight; spsolve fills in on random graphs
    X, _, _ = oracle.di(s, t, n, d=D, tol=1e-15, variant="sop")
    for reorder in (True, False):
        H, *_ = run(s, t, n, 3, [dict(d=D, tol=1e-13)], reorder=reorder)[0]
        assert l1(H, X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
    Xd, _, _ = oracle.di(*csr_dedup(s, t), n, d=D, tol=1e-15, variant="sop")
    H, *_ = run(s, t, n, 2, [dict(d=D, tol=1e-13)], dedup=True)[0]
    assert l1(H, Xd) <= (1e-13 + 1e-15) / (1 - D) + 1e-14


def csr_dedup(s, t):
    k = np.unique(s.astype(np.int64) * (1 << 32) + t.astype(np.int64))
    return (k >> 32).astype(np.int32), (k & 0xFFFFFFFF).astype(np.int32)


@pytest.mark.slow
@pytest.mark.parametrize("asynchronous", [False, True])
def test_c2_partitioned_vs_oracle(asynchronous):
    need_gpu()
    src, dst, n = digen.make("c2", seed=1)
    H, F, st, sts, _ = run(src, dst, n, 2, [dict(d=D, tol=1e-10, variant="sop",
                                                 asynchronous=asynchronous)])[0]
    same_stats(sts)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    assert st["converged"] == 1 and l1(H, Ho) <= 1e-9


def test_async_partitioned_invariants():
    """Asynchronous cycles on 3 ranks: F = B + P.H - H and conservation after 1, 2, 5 cycles
    (every fluid move is atomic, across the exchange as well), and the hub / ragged graph."""
    need_gpu()
    src, dst, n = digen.make("c1", seed=3)
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    outd = np.bincount(src, minlength=n)
    for H, F, st, sts, _ in run(src, dst, n, 3, [dict(d=D, tol=1e-300, variant="sop", max_sweeps=k,
                                                      asynchronous=True) for k in (1, 2, 5)]):
        same_stats(sts)
        assert np.all(F >= 0)
        assert np.abs(F - (B + P @ H - H)).max() <= 1e-15
        cons = F.sum() + (1 - D) * H[outd > 0].sum() + H[outd == 0].sum()
        assert abs(cons - (1 - D)) <= 1e-14
    n = 20000
    rng = np.random.default_rng(7)
    s = rng.integers(0, n, 4 * n).astype(np.int32)
    t = rng.integers(0, n, 4 * n).astype(np.int32)
    s = np.concatenate([s, np.zeros(15000, np.int32)])
    t = np.concatenate([t, np.arange(1, 15001, dtype=np.int32)])
    X, _, _ = oracle.di(s, t, n, d=D, tol=1e-15, variant="sop")
    H, *_ = run(s, t, n, 4, [dict(d=D, tol=1e-13, asynchronous=True)])[0]
    assert l1(H, X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14


def test_invalid_partitioned_arguments(monkeypatch):
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.make("c1")

    def dist_async_flags(r, grp):   # F2 runs asynchronous cycles only
        g = di.Graph(src, dst, n, rank=r, world=2, group=grp)
        try:
            with pytest.raises(di.DIError) as ei:
                g.solve(dist_async=True)
            assert ei.value.status == di.DI_EINVAL and "DI_ASYNC" in str(ei.value)
        finally:
            g.free()

    def no_inbox(r, grp):           # F2 needs the peer-memory inboxes
        g = di.Graph(src, dst, n, rank=r, world=2, group=grp)
        try:
            with pytest.raises(di.DIError) as ei:
                g.solve(asynchronous=True, dist_async=True)
            assert ei.value.status == di.DI_EINVAL and "inbox" in str(ei.value)
            st = g.solve(asynchronous=True)            # the send/recv path still works
            assert st["converged"] == 1 and st["p2p_exchanges"] == 0
        finally:
            g.free()

    from paper_1204_6255_b200.dist import run_local_group
    run_local_group(2, dist_async_flags)
    with di.option("p2p", 0):
        run_local_group(2, no_inbox)
    g = di.Graph(src, dst, n)                          # one GPU: the flag is ignored
    assert g.solve(asynchronous=True, dist_async=True)["converged"] == 1
    g.free()

    def bad_csc(r, grp):
        di.Graph(src, dst, n, rank=r, world=2, group=grp, build_csc=True)

    from paper_1204_6255_b200.dist import run_local_group
    with pytest.raises(di.DIError):
        run_local_group(2, bad_csc)
    with pytest.raises(di.DIError):   # world larger than the group
        grp = di.LocalGroup(2)
        di.Graph(src, dst, n, rank=0, world=3, group=grp)


@pytest.mark.parametrize("asynchronous", [False, True])
def test_nccl_backend_single_rank(asynchronous, monkeypatch):
    """The NCCL backend for real on one GPU: a communicator of one rank (ncclCommInitRank,
    ncclAllReduce, grouped send/recv with no peers) runs the whole partitioned protocol with
    nothing to exchange; C1 to the north_star gate, and the same through a group of one. With
    the option p2p_force = 1 the upload also creates the peer-memory inbox on the one rank (ncclMemAlloc,
    a symmetric ncclCommWindowRegister, the LSA pointer read on the device), and every sweep
    takes the fused path with no peers."""
    need_gpu()
    import paper_1204_6255_b200 as di
    di.set_option("p2p_force", 1)
    try:
        src, dst, n = digen.make("c1", seed=2)
        Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
        nid = di.nccl_unique_id()
        g = di.Graph(src, dst, n, rank=0, world=1, nccl_id=nid)
        assert g.range() == (0, n)
        st = g.solve(d=D, tol=1e-10, asynchronous=asynchronous)
        assert st["converged"] == 1 and st["exchange_entries"] == 0
        assert st["p2p_exchanges"] == st["sweeps"]          # the window exists
        assert l1(g.history().cpu().numpy(), Ho) <= 1e-9
        st = g.solve(d=D, tol=1e-10, asynchronous=asynchronous, exchange="dense")  # one rank: no-op
        assert st["converged"] == 1 and st["dense_exchanges"] == 0
        assert g.residual() <= 1e-10
        g2 = di.Graph(src, dst, n, rank=0, world=1, nccl_id=nid)   # same id: the same communicator
        assert g2.solve(d=D, tol=1e-10, asynchronous=asynchronous)["converged"] == 1
        g.free()
        g2.free()
        g3 = di.Graph(src, dst, n, rank=0, world=1, nccl_id=nid)   # ... also after both were freed
        st = g3.solve(d=D, tol=1e-10, asynchronous=asynchronous)
        assert st["converged"] == 1 and l1(g3.history().cpu().numpy(), Ho) <= 1e-9
        g3.free()
        grp = di.LocalGroup(1)
        g = di.Graph(src, dst, n, rank=0, world=1, group=grp)
        st = g.solve(d=D, tol=1e-10, asynchronous=asynchronous)
        assert st["converged"] == 1
        assert l1(g.history().cpu().numpy(), Ho) <= 1e-9
        g.free()
        grp.free()
    finally:
        di.set_option("p2p_force", 0)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_compact_remote_cold_records(G):
    """The compact remote path of asynchronous partitioned cycles (VERDICT r1 "Next
    round" 4): hot remote targets (the first remote_tier ids of every range) accumulate in the
    compact accumulator and are compacted into 12-B records; pushes to colder remote targets are
    16-B records written by k_cycle straight into the owner's inbox. A small remote_tier forces
    most remote pushes through the cold records. Pins, random graphs with loops and duplicates
    vs the dense solve, C1 to the north_star gate; exchange counters consistent."""
    need_gpu()
    import paper_1204_6255_b200 as di
    with di.option("remote_tier", 3):
        for name, n, links, X in load_pins():
            if n < G:
                continue
            src = np.array([s for s, _ in links], dtype=np.int32)
            dst = np.array([t for _, t in links], dtype=np.int32)
            (H, F, st, sts, _), = run(src, dst, n, G, [dict(d=D, tol=1e-16, asynchronous=True)])
            assert st["converged"] == 1 and l1(H, [float(x) for x in X]) <= 1e-14, name
        for seed in range(15):
            src, dst, n = digen.small_random(seed, n_max=200)
            if n < G:
                continue
            X = defn.solve_dense(src, dst, n, D) if n <= 64 else oracle.di(src, dst, n, d=D, tol=1e-15)[0]
            for H, F, st, sts, _ in run(src, dst, n, G, [dict(d=D, tol=1e-15, variant=v, asynchronous=True)
                                                          for v in ("sop", "cyc")]):
                same_stats(sts)
                assert st["converged"] == 1 and l1(H, X) <= 1e-13 * max(1, n / 64), seed
    src, dst, n = digen.make("c1", seed=1)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    with di.option("remote_tier", 300):
        res = run(src, dst, n, G, [dict(d=D, tol=1e-10, asynchronous=True),
                                   dict(d=D, tol=1e-10, asynchronous=True, profile=True)])
    for H, F, st, sts, ranges in res:
        same_stats(sts)
        assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
        assert l1(H, Ho) <= 1e-9
        assert all(s["exchange_cold"] > 0 and s["exchange_entries"] > 0 for s in sts)
        for s in sts:
            assert s["exchange_bytes"] == 12 * s["exchange_entries"] + 16 * s["exchange_cold"]
            assert s["p2p_exchanges"] == s["sweeps"]


@pytest.mark.parametrize("G,parts", [(2, 2), (4, 3), (8, 4)])
def test_dist_parts(G, parts):
    """Option dist_parts: each rank's asynchronous cycle runs in `parts` launches over
    consecutive claim windows of its tiles, the exchange after each, so remote fluid arrives within
    the cycle. Pins, random graphs with loops and duplicates vs the dense solve, and C1 to the
    north_star gate against the oracle, with the compact remote path (a small remote tier: cold
    records) and the plain one."""
    need_gpu()
    import paper_1204_6255_b200 as di
    with di.option("dist_parts", parts), di.option("remote_tier", 5):
        for name, n, links, X in load_pins():
            if n < G:
                continue
            src = np.array([s for s, _ in links], dtype=np.int32)
            dst = np.array([t for _, t in links], dtype=np.int32)
            (H, F, st, sts, _), = run(src, dst, n, G, [dict(d=D, tol=1e-16, asynchronous=True)])
            assert st["converged"] == 1 and l1(H, [float(x) for x in X]) <= 1e-14, (name, st, l1(H, [float(x) for x in X]))
        for seed in range(8):
            src, dst, n = digen.small_random(seed, n_max=3000 if seed % 2 else 200)
            if n < G:
                continue
            X = defn.solve_dense(src, dst, n, D) if n <= 64 else oracle.di(src, dst, n, d=D, tol=1e-15)[0]
            for H, F, st, sts, _ in run(src, dst, n, G, [dict(d=D, tol=1e-15, variant=v, asynchronous=True)
                                                          for v in ("sop", "cyc")]):
                same_stats(sts)
                assert st["converged"] == 1 and l1(H, X) <= 1e-13 * max(1, n / 64), seed
    src, dst, n = digen.make("c1", seed=2)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    for rt in (0, 300):
        with di.option("dist_parts", parts), di.option("remote_tier", rt):
            (H, F, st, sts, _), = run(src, dst, n, G, [dict(d=D, tol=1e-10, asynchronous=True)])
        same_stats(sts)
        assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
        assert l1(H, Ho) <= 1e-9
