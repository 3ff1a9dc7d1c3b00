"""GPU D-iteration solves vs the oracle and vs properties that hold at any size (T1, T2, T7-T10)."""
import numpy as np
import pytest

import digen
import oracle
from conftest import load_pins
from gpu_util import l1, need_gpu, upload, warm_count, warm_shift
from oracle import definition as defn

pytestmark = pytest.mark.gpu
D = 0.85
PINS = load_pins()


@pytest.mark.parametrize("variant", ["sop", "cyc"])
def test_exact_pins(variant):
    need_gpu()
    for name, n, links, X in PINS:
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        g = upload(src, dst, n)
        st = g.solve(d=D, tol=1e-16, variant=variant)
        assert st["converged"] == 1, (name, st)
        H = g.history().cpu().numpy()
        assert l1(H, [float(x) for x in X]) <= 1e-14, (name, H)
        g.free()


MODES = ["push", "pull", "auto"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("d", [0.5, 0.85, 0.95])
def test_random_vs_dense(d, mode):
    need_gpu()
    for seed in range(60):
        src, dst, n = digen.small_random(seed)
        X = defn.solve_dense(src, dst, n, d)
        g = upload(src, dst, n, build_csc=True)
        for variant in ("sop", "cyc"):
            st = g.solve(d=d, tol=1e-15, variant=variant, mode=mode)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= 1e-13, (seed, variant)
        g.free()


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("variant", ["sop", "cyc"])
@pytest.mark.parametrize("name,seed", [("c1", 1), ("c1", 2), ("c1", 3), ("c2", 1)])
def test_north_star_parity(name, seed, variant, mode):
    """T10: ||H_gpu - H_oracle||_1 <= 1e-9, both run to ||F||_1 <= 1e-10 (north_star), and
    <= 1e-10/(1-d) + 1e-13/(1-d) against the tight (1e-13) oracle run (reading G19)."""
    need_gpu()
    src, dst, n = digen.make(name, seed=seed)
    g = upload(src, dst, n, build_csc=True)
    st = g.solve(d=D, tol=1e-10, variant=variant, mode=mode)
    if mode == "pull":
        assert st["pull_sweeps"] == st["sweeps"]
    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
    H = g.history().cpu().numpy()
    Ho, _, sto = oracle.di(src, dst, n, d=D, tol=1e-10, variant=variant)
    assert l1(H, Ho) <= 1e-9
    Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant=variant)
    assert l1(H, Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D)
    # accounting: eq-iter = link diffusions / L
    assert abs(st["equivalent_iterations"] - st["link_diffusions"] / len(src)) < 1e-12
    g.free()


@pytest.mark.parametrize("blocks", [2, 3, 8])
def test_block_ordered_vs_exact(blocks):
    """Block-ordered cycles (F1): exact pins, random graphs with loops/duplicates vs the
    dense solve, the invariant F = B + P.H - H at arbitrary stops (also mid-cycle)."""
    need_gpu()
    for name, n, links, X in PINS:
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            st = g.solve(d=D, tol=1e-16, variant=variant, blocks=blocks)
            assert st["converged"] == 1, (name, st)
            assert l1(g.history().cpu().numpy(), [float(x) for x in X]) <= 1e-14, name
        g.free()
    for seed in range(40):
        src, dst, n = digen.small_random(seed, n_max=3000 if seed % 4 == 0 else 64)
        X = defn.solve_dense(src, dst, n, D) if n <= 64 else defn.solve_sparse(src, dst, n, D)
        P = defn.sparse_P(src, dst, n, D)
        B = defn.uniform_B(n, D)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            st = g.solve(d=D, tol=1e-15, variant=variant, blocks=blocks)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= 1e-13 * max(1, n / 64), (seed, variant)
            g.solve(d=D, tol=1e-300, variant=variant, blocks=blocks, max_sweeps=2)
            H = g.history().cpu().numpy()
            _, F = g.residual(return_F=True)
            F = F.cpu().numpy()
            assert np.all(F >= 0) and np.abs(F - (B + P @ H - H)).max() <= 1e-15
        g.free()


@pytest.mark.parametrize("blocks", [4, 16])
@pytest.mark.parametrize("name,seed", [("c1", 1), ("c2", 1)])
def test_block_ordered_north_star(name, seed, blocks):
    """T10 for block-ordered cycles, and the point of F1: fewer link diffusions than the bulk
    sweep (closer to the paper's sequential cycle), within the same tolerance."""
    need_gpu()
    src, dst, n = digen.make(name, seed=seed)
    g = upload(src, dst, n)
    st = g.solve(d=D, tol=1e-10, variant="sop", blocks=blocks, trace=True)
    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
    H = g.history().cpu().numpy()
    Ho, _, sto = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    assert l1(H, Ho) <= 1e-9
    Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant="sop")
    assert l1(H, Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D)
    log = g.sweep_log()
    assert len(log["r"]) == st["sweeps"] and log["links"].sum() == st["link_diffusions"]
    st1 = g.solve(d=D, tol=1e-10, variant="sop")
    assert st["link_diffusions"] < st1["link_diffusions"]
    assert st["sweeps"] < st1["sweeps"]
    g.free()


@pytest.mark.parametrize("blocks,mode", [(1, "push"), (1, "auto"), (8, "push")])
def test_graph_loop(blocks, mode):
    """DI_GRAPH_LOOP (the sweep loop as one CUDA graph with a device-side while node) gives the
    same iterates as the host-driven loop: same sweeps and link diffusions, H within rounding of
    the fp64 atomics; max_sweeps stops it exactly; pins and the north_star gate hold."""
    need_gpu()
    import paper_1204_6255_b200 as di
    for name in ("c1", "c2"):
        src, dst, n = digen.make(name, seed=1)
        g = upload(src, dst, n, build_csc=True)
        st0 = g.solve(d=D, tol=1e-10, blocks=blocks, mode=mode)
        H0 = g.history().cpu().numpy()
        st1 = g.solve(d=D, tol=1e-10, blocks=blocks, mode=mode, graph_loop=True)
        H1 = g.history().cpu().numpy()
        assert st1["converged"] == 1 and st1["residual_l1"] <= 1e-10
        # fp64 atomics make the iterates order-nondeterministic in the last bits, which can flip a
        # threshold test: same sweeps +-1 and link diffusions within 0.1 %
        assert abs(st1["sweeps"] - st0["sweeps"]) <= 1
        assert abs(st1["link_diffusions"] - st0["link_diffusions"]) <= 1e-3 * st0["link_diffusions"]
        assert l1(H0, H1) <= 2e-10 / (1 - D)
        Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
        assert l1(H1, Ho) <= 1e-9
        st2 = g.solve(d=D, tol=1e-10, blocks=blocks, mode=mode, graph_loop=True, max_sweeps=7)
        assert st2["status"] == di.DI_NOT_CONVERGED and st2["sweeps"] == 7
        g.free()
    for pname, n, links, X in PINS:
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        g = upload(src, dst, n, build_csc=True)
        st = g.solve(d=D, tol=1e-16, blocks=blocks, mode=mode, graph_loop=True)
        assert st["converged"] == 1
        assert l1(g.history().cpu().numpy(), [float(x) for x in X]) <= 1e-14, pname
        g.free()


@pytest.mark.parametrize("graph_loop", [False, True])
def test_async_cycles(graph_loop):
    """DI_ASYNC (one persistent kernel per cycle, live F taken by atomic exchange, paper's cyclic
    order up to the grid's concurrency): exact pins, random graphs with loops/duplicates vs the
    dense solve, F = B + P.H - H and conservation at arbitrary stops, north_star gate on C1 and
    C2 for DI-SOP and DI-CYC, ragged sizes around the tile and hub rows above the chunk size."""
    need_gpu()
    import paper_1204_6255_b200 as di
    kw = dict(asynchronous=True, graph_loop=graph_loop)
    for name, n, links, X in PINS:
        src = np.array([s for s, _ in links], dtype=np.int32)
        dst = np.array([t for _, t in links], dtype=np.int32)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            st = g.solve(d=D, tol=1e-16, variant=variant, **kw)
            assert st["converged"] == 1, (name, st)
            assert l1(g.history().cpu().numpy(), [float(x) for x in X]) <= 1e-14, name
        g.free()
    for seed in range(40):
        src, dst, n = digen.small_random(seed, n_max=3000 if seed % 4 == 0 else 64)
        X = defn.solve_dense(src, dst, n, D) if n <= 64 else defn.solve_sparse(src, dst, n, D)
        P = defn.sparse_P(src, dst, n, D)
        B = defn.uniform_B(n, D)
        out = np.bincount(src, minlength=n)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            st = g.solve(d=D, tol=1e-15, variant=variant, **kw)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= 1e-13 * max(1, n / 64), (seed, variant)
            for k in (1, 3):
                st = g.solve(d=D, tol=1e-300, variant=variant, max_sweeps=k, **kw)
                # a cycle in (dynamic) node order can drain a small graph completely (F == 0)
                assert (st["status"] == di.DI_NOT_CONVERGED and st["sweeps"] == k) or \
                       (st["status"] == di.DI_OK and st["residual_l1"] == 0.0 and st["sweeps"] <= k)
                H = g.history().cpu().numpy()
                _, F = g.residual(return_F=True)
                F = F.cpu().numpy()
                assert np.all(F >= 0) and np.abs(F - (B + P @ H - H)).max() <= 1e-15
                cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
                assert abs(cons - (1 - D)) <= 1e-14
        g.free()
    for name, seed in (("c1", 1), ("c1", 2), ("c2", 1)):
        src, dst, n = digen.make(name, seed=seed)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            st = g.solve(d=D, tol=1e-10, variant=variant, trace=True, **kw)
            assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
            H = g.history().cpu().numpy()
            Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant=variant)
            assert l1(H, Ho) <= 1e-9, (name, variant)
            Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant=variant)
            assert l1(H, Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D)
            if not graph_loop:
                log = g.sweep_log()
                assert len(log["r"]) == st["sweeps"] and log["links"].sum() == st["link_diffusions"]
        g.free()
    for n in (1, 1023, 1025, 20000):
        rng = np.random.default_rng(n)
        src = rng.integers(0, n, 4 * n).astype(np.int32)
        dst = rng.integers(0, n, 4 * n).astype(np.int32)
        if n == 20000:   # hub rows of 15000 and 3000 links (several 1024-link chunks)
            src = np.concatenate([src, np.zeros(15000, np.int32), np.full(3000, 5, np.int32)])
            dst = np.concatenate([dst, np.arange(1, 15001, dtype=np.int32), np.arange(6, 3006, dtype=np.int32)])
        X, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant="sop")
        g = upload(src, dst, n)
        st = g.solve(d=D, tol=1e-13, **kw)
        assert st["converged"] == 1
        assert l1(g.history().cpu().numpy(), X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
        g.free()
    g = di.Graph(np.zeros(0, np.int32), np.zeros(0, np.int32), 3000)
    st = g.solve(d=D, tol=1e-12, **kw)
    assert st["converged"] == 1 and st["sweeps"] == 1
    g.free()
    # resume after max_sweeps, custom B, the paper's stop
    src, dst, n = digen.make("c1", seed=3)
    g = upload(src, dst, n)
    rng = np.random.default_rng(9)
    Bc = rng.random(n) * (1 - D) / n * 2
    st = g.solve(d=D, tol=1e-12, B=Bc, max_sweeps=4, **kw)
    assert st["status"] == di.DI_NOT_CONVERGED and st["sweeps"] == 4
    st = g.solve(d=D, tol=1e-12, B=Bc, resume=True, **kw)
    assert st["converged"] == 1
    assert l1(g.history().cpu().numpy(), defn.solve_sparse(src, dst, n, D, B=Bc)) <= 1e-12 / (1 - D)
    st = g.solve(d=D, tol=1.0 / n, paper_error=True, **kw)
    assert st["converged"] == 1 and st["error_estimate"] <= 1.0 / n
    g.free()
    # skewed in-degrees on a power-of-two stripe length: the replicated hot accumulators path
    # (N = 4096 * 8, three targets with 4 %, 2 %, 1 % of all links)
    n = 4096 * 8
    rng = np.random.default_rng(11)
    src = rng.integers(0, n, 6 * n).astype(np.int32)
    dst = rng.integers(0, n, 6 * n).astype(np.int32)
    m = len(src)
    for hub, share in ((77, 0.04), (5000, 0.02), (123, 0.01)):
        k = int(share * m)
        src = np.concatenate([src, rng.integers(0, n, k).astype(np.int32)])
        dst = np.concatenate([dst, np.full(k, hub, np.int32)])
    g = upload(src, dst, n)
    for variant in ("sop", "cyc"):
        X, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant=variant)
        st = g.solve(d=D, tol=1e-13, variant=variant, **kw)
        assert st["converged"] == 1
        assert l1(g.history().cpu().numpy(), X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
    g.free()
    # hot targets that are also hubs (R-MAT-like): rows of 30000 / 9000 links (> kHubMin) are
    # pushed as hub items (async.cu); one hub row carries a self-loop (LOOPS path)
    rng = np.random.default_rng(12)
    src = rng.integers(0, n, 6 * n).astype(np.int32)
    dst = rng.integers(0, n, 6 * n).astype(np.int32)
    m = len(src)
    for hub, share, out in ((77, 0.04, 30000), (5000, 0.02, 9000), (123, 0.01, 100)):
        k = int(share * m)
        tgt = rng.choice(n, out, replace=False).astype(np.int32)
        src = np.concatenate([src, rng.integers(0, n, k).astype(np.int32), np.full(out, hub, np.int32)])
        dst = np.concatenate([dst, np.full(k, hub, np.int32), tgt])
    src = np.concatenate([src, np.array([77], np.int32)])
    dst = np.concatenate([dst, np.array([77], np.int32)])
    g = upload(src, dst, n)
    for variant in ("sop", "cyc"):
        X, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant=variant)
        for rep in range(2):   # a second solve on the same graph: hub flags carry over
            st = g.solve(d=D, tol=1e-13, variant=variant, **kw)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
    g.free()


def test_threshold_scale():
    """F4: di_set_threshold_scale. alpha = 1 is the paper's rule (same solve as the default);
    other alphas reach the same fixed point within the north_star gate; alpha <= 0 is refused."""
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.make("c1", seed=1)
    Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant="sop")
    g = upload(src, dst, n)
    st0 = g.solve(d=D, tol=1e-10, variant="sop")
    for alpha in (1.0, 0.5, 2.0, 4.0):
        g.set_threshold_scale(alpha)
        for kw in (dict(), dict(asynchronous=True), dict(blocks=4)):
            st = g.solve(d=D, tol=1e-10, variant="sop", **kw)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D)
            if alpha == 1.0 and not kw:
                assert abs(st["sweeps"] - st0["sweeps"]) <= 1
    with pytest.raises(di.DIError):
        g.set_threshold_scale(0.0)
    g.free()


@pytest.mark.parametrize("mode", MODES)
def test_invariants_mid_solve(mode):
    """T8: at any stopping point F = B + P.H - H, F >= 0, conservation, sum F non-increasing."""
    need_gpu()
    for seed in range(20):
        src, dst, n = digen.small_random(seed, n_max=64)
        P = defn.dense_P(src, dst, n, D)
        B = defn.uniform_B(n, D)
        out = np.bincount(src, minlength=n)
        g = upload(src, dst, n, build_csc=True)
        for variant in ("sop", "cyc"):
            prev = np.inf
            for k in (1, 2, 3, 5, 8):
                g.solve(d=D, tol=1e-300, variant=variant, max_sweeps=k, mode=mode)
                H = g.history().cpu().numpy()
                r, F = g.residual(return_F=True)
                F = F.cpu().numpy()
                assert np.all(F >= 0)
                assert np.abs(F - (B + P @ H - H)).max() <= 1e-15
                cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
                assert abs(cons - (1 - D)) <= 1e-14
                assert F.sum() <= prev + 1e-17
                prev = F.sum()
        g.free()


@pytest.mark.parametrize("mode", MODES)
def test_bulk_cyc_neumann_gpu(mode):
    """T7: bulk DI-CYC without loops: F_n = P^n B and H_n = sum_{k<n} P^k B after n sweeps."""
    need_gpu()
    src, dst, n = digen.make("c1")
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    g = upload(src, dst, n, build_csc=True)
    Fn, Hn = B.copy(), np.zeros(n)
    for k in range(1, 11):
        g.solve(d=D, tol=1e-300, variant="cyc", max_sweeps=k, mode=mode)
        Hn = Hn + Fn
        Fn = P @ Fn
        _, F = g.residual(return_F=True)
        F = F.cpu().numpy()
        H = g.history().cpu().numpy()
        nz = Fn > 0
        assert np.array_equal(F > 0, nz)
        assert np.max(np.abs(F[nz] - Fn[nz]) / Fn[nz]) <= 1e-13
        assert np.max(np.abs(H - Hn) / np.maximum(Hn, 1e-300)) <= 1e-13
    g.free()


@pytest.mark.parametrize("mode", MODES)
def test_closure_drainage_gpu(mode):
    """T9: nodes of E at depth <= t hold exactly 0.0 after t+1 bulk DI-CYC sweeps."""
    need_gpu()
    for seed in range(30):
        src, dst, n = digen.dag_fringe(seed)
        depth = digen.closure(src, dst, n)
        g = upload(src, dst, n, build_csc=True)
        for t in range(6):
            g.solve(d=D, tol=1e-300, variant="cyc", max_sweeps=t + 1, mode=mode)
            _, F = g.residual(return_F=True)
            F = F.cpu().numpy()
            drained = (depth >= 0) & (depth <= t)
            assert np.all(F[drained] == 0.0), (seed, t)
        g.free()


def test_resume_and_not_converged():
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.make("c1")
    g = upload(src, dst, n)
    st = g.solve(d=D, tol=1e-10, variant="sop", max_sweeps=5)
    assert st["status"] == di.DI_NOT_CONVERGED and st["sweeps"] == 5
    st2 = g.solve(d=D, tol=1e-10, variant="sop", resume=True)
    assert st2["converged"] == 1
    H = g.history().cpu().numpy()
    X = defn.solve_sparse(src, dst, n, D)
    assert l1(H, X) <= 1e-10 / (1 - D)
    with pytest.raises(di.DIError):
        g.solve(d=1.0)
    with pytest.raises(di.DIError):
        g.solve(tol=0.0)
    g.free()


def test_edge_cases():
    need_gpu()
    import paper_1204_6255_b200 as di
    # all dangling, L = 0: one sweep absorbs everything, X = (1-d)/N
    g = di.Graph(np.zeros(0, np.int32), np.zeros(0, np.int32), 3000)
    st = g.solve(d=D, tol=1e-12)
    assert st["converged"] == 1 and st["sweeps"] == 1
    assert np.allclose(g.history().cpu().numpy(), (1 - D) / 3000, rtol=0, atol=1e-18)
    g.free()
    # N around the select tile size (1024 nodes per tile): ragged tails; hub rows > chunk sizes
    for n in (1, 1023, 1024, 1025, 4097, 20000):
        rng = np.random.default_rng(n)
        m = 4 * n
        src = rng.integers(0, n, m).astype(np.int32)
        dst = rng.integers(0, n, m).astype(np.int32)
        if n == 20000:   # one out-hub (push bin C) and one in-hub (pull bin P3)
            src = np.concatenate([src, np.zeros(15000, np.int32), np.arange(1, 12001, dtype=np.int32)])
            dst = np.concatenate([dst, np.arange(1, 15001, dtype=np.int32), np.full(12000, 7, np.int32)])
        g = upload(src, dst, n, build_csc=True)
        # reference: the (pinned) sequential oracle run tight; spsolve fills in on random graphs
        X, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant="sop")
        for variant, mode in (("sop", "push"), ("cyc", "push"), ("sop", "pull"), ("sop", "auto")):
            st = g.solve(d=D, tol=1e-13, variant=variant, mode=mode)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14
        g.free()


def test_custom_B_and_paper_stop():
    need_gpu()
    src, dst, n = digen.make("c1")
    rng = np.random.default_rng(5)
    B = rng.random(n) * (1 - D) / n * 2
    g = upload(src, dst, n)
    st = g.solve(d=D, tol=1e-12, B=B)
    X = defn.solve_sparse(src, dst, n, D, B=B)
    assert l1(g.history().cpu().numpy(), X) <= 1e-12 / (1 - D)
    st = g.solve(d=D, tol=1.0 / n, paper_error=True)
    assert st["converged"] == 1 and st["error_estimate"] <= 1.0 / n
    Ho, _, sto = oracle.di(src, dst, n, d=D, tol=1.0 / n, variant="sop", paper_stop=True)
    X = defn.solve_sparse(src, dst, n, D)
    H = g.history().cpu().numpy()
    assert l1(H / H.sum(), X / X.sum()) <= 2 * st["error_estimate"]
    g.free()


def test_trace_log():
    need_gpu()
    src, dst, n = digen.make("c1")
    g = upload(src, dst, n, build_csc=True)
    st = g.solve(d=D, tol=1e-10, trace=True, profile=True, mode="auto")
    log = g.sweep_log()
    assert log["mode"].sum() == st["pull_sweeps"] > 0
    assert np.all((log["links"] > int(0.35 * len(src))) == (log["mode"] == 1))
    assert len(log["r"]) == st["sweeps"]
    assert log["links"].sum() == st["link_diffusions"] and log["selected"].sum() == st["selected_total"]
    assert np.all(np.diff(log["r"]) <= 1e-18)                       # sum F non-increasing
    assert st["push_ms"] > 0 and st["select_ms"] > 0
    g.free()


@pytest.mark.slow
def test_c3_async_vs_oracle():
    """The north_star gate at C3's full size (host-block graph, 8.4M nodes, ~99M links, Zipf hot
    targets: replicated accumulators on), the bench's launch configuration against the sequential
    CPU oracle, both to ||F||_1 <= 1e-10."""
    need_gpu()
    src, dst, n = digen.make("c3")
    g = upload(src, dst, n)
    st = g.solve(d=D, tol=1e-10, variant="sop", asynchronous=True, graph_loop=True)
    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
    H = g.history().cpu().numpy()
    g.free()
    Ho, _, sto = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    assert l1(H, Ho) <= 1e-9


@pytest.mark.slow
def test_c4_full_size_properties():
    """C4 at full size, first in the bench's launch configuration (asynchronous cycles in the
    device-side graph loop), then bulk sweeps with the push/pull choice: the north_star gate
    against the sequential CPU oracle (both to ||F||_1 <= 1e-10), converged residual, sampled
    invariant F_i = B_i + (P.H)_i - H_i on 2000 nodes, conservation, and
    ||X - H||_1 <= ||F||_1/(1-d) by construction."""
    need_gpu()
    src, dst, n = digen.make("c4")
    g = upload(src, dst, n, build_csc=True)
    rng = np.random.default_rng(0)
    sample = rng.choice(n, 2000, replace=False)
    out = np.bincount(src, minlength=n).astype(np.float64)
    insample = np.isin(dst, sample)
    Ho = None
    for kw in (dict(asynchronous=True, graph_loop=True), dict(mode="auto")):
        st = g.solve(d=D, tol=1e-10, variant="sop", **kw)
        assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
        if "mode" in kw:
            assert 0 < st["pull_sweeps"] < st["sweeps"]
        H = g.history().cpu().numpy()
        if Ho is None:   # the north_star gate on the bench's workload and launch configuration
            Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
        assert l1(H, Ho) <= 1e-9, kw
        _, F = g.residual(return_F=True)
        F = F.cpu().numpy()
        assert np.all(F >= 0) and np.all(H >= 0)
        ph = np.zeros(n)
        np.add.at(ph, dst[insample], D * H[src[insample]] / out[src[insample]])
        resid = (1 - D) / n + ph[sample] - H[sample]
        assert np.max(np.abs(resid - F[sample])) <= 1e-15, kw
        cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
        assert abs(cons - (1 - D)) <= 1e-12, kw
    g.free()
    # the partitioned path at the same size: 4 emulated ranks on this GPU (fused peer-memory
    # exchange; then asynchronous multi-GPU cycles), the same gate against the same oracle run
    import torch
    import paper_1204_6255_b200 as di
    from paper_1204_6255_b200.dist import assemble, run_local_group
    s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()

    def rank(r, grp):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            gr = di.Graph(s_d, t_d, n, rank=r, world=4, group=grp, stream=stream)
            out_ = []
            for kw in (dict(asynchronous=True), dict(asynchronous=True, dist_async=True)):
                st = gr.solve(d=D, tol=1e-10, variant="sop", **kw)
                out_.append((gr.history().cpu().numpy(), st))
            rg = (gr.lo, gr.hi)
            gr.free()
        return rg, out_

    res = run_local_group(4, rank)
    for k in range(2):
        H = assemble([o[k][0] for _, o in res], [rg for rg, _ in res], n)
        assert res[0][1][k][1]["converged"] == 1
        assert l1(H, Ho) <= 1e-9, k


@pytest.mark.parametrize("axis", ["transpose", "loops"])
def test_paper_axes_c2_async_vs_oracle(axis):
    """F3's paper axes at C2's full size, on the bench's path (asynchronous cycles in the
    device-side graph loop): Dataset 1bis is P^T (every link reversed) and Dataset 1
    has O/N = 0.204 self-loop nodes (Table 1; fold P:259-263, reading G6), here 20 % of
    the nodes with out-links get one self-loop (the LOOPS instantiation of k_cycle). North_star
    gate against the sequential CPU oracle (both to ||F||_1 <= 1e-10), and against the tight
    oracle run (G19); DI-SOP and DI-CYC; the bulk push sweep too."""
    need_gpu()
    src, dst, n = digen.make("c2")
    if axis == "transpose":
        src, dst = digen.transpose(src, dst)
    else:
        src, dst = digen.add_self_loops(src, dst, n, frac=0.2)
        assert digen.stats(src, dst, n)["o_over_n"] > 0.15
    g = upload(src, dst, n)
    for variant in ("sop", "cyc"):
        Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant=variant)
        Ht, _, _ = oracle.di(src, dst, n, d=D, tol=1e-13, variant=variant)
        for kw in (dict(asynchronous=True, graph_loop=True), dict()):
            st = g.solve(d=D, tol=1e-10, variant=variant, **kw)
            assert st["converged"] == 1 and st["residual_l1"] <= 1e-10, (axis, variant, kw)
            H = g.history().cpu().numpy()
            assert l1(H, Ho) <= 1e-9, (axis, variant, kw)
            assert l1(H, Ht) <= 1e-10 / (1 - D) + 1e-13 / (1 - D), (axis, variant, kw)
    g.free()


def _skewed_hub_graph(seed, n=4096 * 8, self_loop_on_hot=True):
    """Targets with 4 %, 2 %, 1 % of all links (replicated accumulators on) that are also hub rows
    of 30000 / 9000 / 100 links; one hot hub row carries a self-loop (fold, G6)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 6 * n).astype(np.int32)
    dst = rng.integers(0, n, 6 * n).astype(np.int32)
    m = len(src)
    for hub, share, out in ((77, 0.04, 30000), (5000, 0.02, 9000), (123, 0.01, 100)):
        k = int(share * m)
        tgt = rng.choice(n, out, replace=False).astype(np.int32)
        src = np.concatenate([src, rng.integers(0, n, k).astype(np.int32), np.full(out, hub, np.int32)])
        dst = np.concatenate([dst, np.full(k, hub, np.int32), tgt])
    if self_loop_on_hot:
        src = np.concatenate([src, np.array([77, 5000], np.int32)])
        dst = np.concatenate([dst, np.array([77, 5000], np.int32)])
    return src, dst, n


@pytest.mark.parametrize("kw", [dict(), dict(mode="auto"), dict(blocks=8), dict(mode="pull")],
                         ids=["bulk_push", "auto", "blocks8", "pull"])
def test_hot_accumulators_every_schedule(kw):
    """The replicated hot accumulators are folded by every push schedule (bulk k_push, the DI_AUTO
    push/pull mix, block-ordered sub-sweeps), not only by the asynchronous cycle: skewed in-degrees
    (hot placement on), hot targets that are hub rows, self-loops on hot hubs."""
    need_gpu()
    src, dst, n = _skewed_hub_graph(21)
    g = upload(src, dst, n, build_csc=True)
    for variant in ("sop", "cyc"):
        X, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant=variant)
        for rep in range(2):
            st = g.solve(d=D, tol=1e-13, variant=variant, **kw)
            assert st["converged"] == 1
            assert l1(g.history().cpu().numpy(), X) <= (1e-13 + 1e-15) / (1 - D) + 1e-14, (variant, rep)
    g.free()


def test_hot_accumulators_pi_push():
    """PI' (push comparator) scatters through the same replicated accumulators (k_pi_fold): on the
    skewed hub graph with self-loops it matches the oracle's PI' loop and the normalised fixed
    point."""
    need_gpu()
    src, dst, n = _skewed_hub_graph(22)
    g = upload(src, dst, n, build_csc=True)
    target = 1e-12
    st = g.solve(d=D, tol=target, variant="pi_push")
    x = g.history().cpu().numpy()
    xo, sto = oracle.pi_col(src, dst, n, d=D, target=target)
    assert st["converged"] == 1 and abs(st["sweeps"] - sto["cycles"]) <= 1
    if st["sweeps"] == sto["cycles"]:
        assert l1(x, xo) <= 1e-12
    # (a sparse direct solve of this graph fills in catastrophically: the pinned oracle at 1e-15)
    Xs, _, _ = oracle.di(src, dst, n, d=D, tol=1e-15, variant="sop")
    assert l1(x, Xs / Xs.sum()) <= 1e-10
    g.free()


@pytest.mark.parametrize("warm", [0, 128, 4032, 60000])
def test_warm_tier(warm):
    """Warm tier (option warm): k_cycle accumulates its pushes to the `warm` hottest
    ids in each CTA's shared memory and flushes them into F when the CTA leaves the cycle — a delay
    of that fluid to the cycle's end, which any diffusion order allows. Placement: the
    warm ranks one every 2^s ids after the 64 hot ids (checked through the relabelling); 60000 is
    above what fits in shared memory, so ids past the capacity take the plain RED. The gate against
    the oracle on C2 (R-MAT, skewed), a skewed graph with hub rows and a self-loop on a hot node
    (LOOPS instantiation), DI-SOP and DI-CYC, host loop and graph loop; with cold bins forced on the
    tier is off (graph_build.cu) and the same gate holds."""
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.make("c2")
    rng = np.random.default_rng(12)
    n2 = 4096 * 16
    s2 = rng.integers(0, n2, 6 * n2).astype(np.int32)
    t2 = rng.integers(0, n2, 6 * n2).astype(np.int32)
    m = len(s2)
    for hub, share, out in ((77, 0.04, 30000), (5000, 0.02, 9000), (123, 0.01, 100)):
        k = int(share * m)
        tgt = rng.choice(n2, out, replace=False).astype(np.int32)
        s2 = np.concatenate([s2, rng.integers(0, n2, k).astype(np.int32), np.full(out, hub, np.int32), [77]])
        t2 = np.concatenate([t2, np.full(k, hub, np.int32), tgt, [77]]).astype(np.int32)
    s2 = s2.astype(np.int32)
    for (s_, t_, nn) in ((src, dst, n), (s2, t2, n2)):
        indeg = np.bincount(t_, minlength=nn)
        for cold in (0, 1):
            with di.option("warm", warm), di.option("cold_bins", cold), di.option("cold_tier", nn // 8):
                g = upload(s_, t_, nn)
            if not cold and warm_count(indeg, len(s_), nn, warm, hot=64):   # hot, then warm every S ids
                old_of = g.test_perm()
                ranked = np.argsort(-indeg, kind="stable").astype(np.int32)
                sh = warm_shift(warm, nn // 8 if cold else nn - 64)
                assert np.array_equal(old_of[:64], ranked[:64])
                assert np.array_equal(old_of[64 + (np.arange(warm) << sh)], ranked[64:64 + warm])
            for variant in ("sop", "cyc"):
                Ho, _, _ = oracle.di(s_, t_, nn, d=D, tol=1e-10, variant=variant)
                for graph_loop in (False, True):
                    st = g.solve(d=D, tol=1e-10, variant=variant, asynchronous=True, graph_loop=graph_loop)
                    assert st["converged"] == 1 and st["residual_l1"] <= 1e-10
                    assert l1(g.history().cpu().numpy(), Ho) <= 1e-9, (nn, cold, variant, graph_loop)
            if nn == n2:   # stopped after k cycles: the flushed accumulators leave F = B + P.H - H
                P = defn.sparse_P(s_, t_, nn, D)
                B = defn.uniform_B(nn, D)
                out = np.bincount(s_, minlength=nn)
                for k in (1, 2, 5):
                    st = g.solve(d=D, tol=1e-300, max_sweeps=k, asynchronous=True)
                    assert st["sweeps"] == k
                    H = g.history().cpu().numpy()
                    _, F = g.residual(return_F=True)
                    F = F.cpu().numpy()
                    assert np.all(F >= 0) and np.abs(F - (B + P @ H - H)).max() <= 1e-15, (warm, cold, k)
                    cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
                    assert abs(cons - (1 - D)) <= 1e-14, (warm, cold, k)
            g.free()
