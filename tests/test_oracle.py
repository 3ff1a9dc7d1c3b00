"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each test checks the oracle against something the paper or mathematics fixes:
exact rationals (tests/golden/pins.txt), a dense / sparse library solve of
(I - P) X = B (§1), the invariant F = B + P.H - H, the error
bound ||X - H||_1 <= ||F||_1/(1-d), mass conservation, Neumann partial sums for
bulk DI-CYC, closure drainage and the starvation cases of reading G5.
"""
from fractions import Fraction

import numpy as np
import pytest

import digen
import oracle
from oracle import definition as defn
from conftest import load_pins

PINS = load_pins()
D = 0.85


def l1(a, b):
    return float(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)).sum())


def links_arrays(links):
    src = np.array([s for s, _ in links], dtype=np.int32)
    dst = np.array([t for _, t in links], dtype=np.int32)
    return src, dst


# ------------------------------------------------------------------ exact pins
@pytest.mark.parametrize("pin", PINS, ids=[p[0] for p in PINS])
def test_exact_definition(pin):
    """The fixture rationals solve X = P.X + B exactly (d = 17/20), and satisfy the mass identity."""
    name, n, links, X = pin
    d = Fraction(17, 20)
    assert defn.solve_exact(links, n, d) == X
    out = [0] * n
    for s, _ in links:
        out[s] += 1
    dang = sum(X[i] for i in range(n) if out[i] == 0)
    assert (1 - d) * sum(X) + d * dang == 1 - d


@pytest.mark.parametrize("pin", PINS, ids=[p[0] for p in PINS])
@pytest.mark.parametrize("variant", ["cyc", "sop"])
def test_di_exact_pins(pin, variant):
    name, n, links, X = pin
    src, dst = links_arrays(links)
    Xf = np.array([float(x) for x in X])
    for bulk in (False, True):
        fn = oracle.bulk_di if bulk else oracle.di
        H, F, st = fn(src, dst, n, d=D, tol=1e-16, variant=variant)
        assert st["converged"] == 1
        assert l1(H, Xf) <= 1e-14, (name, bulk, H, Xf)
        assert F.sum() <= 1e-16


@pytest.mark.parametrize("pin", PINS, ids=[p[0] for p in PINS])
def test_gs_pi_exact_pins(pin):
    name, n, links, X = pin
    src, dst = links_arrays(links)
    Xf = np.array([float(x) for x in X])
    x, st = oracle.gs(src, dst, n, d=D, target=1e-15)
    assert st["converged"] == 1 and l1(x, Xf) <= 1e-14
    Xn = Xf / Xf.sum()
    for fn in (oracle.pi, oracle.pi_col):
        x, st = fn(src, dst, n, d=D, target=1e-15)
        assert st["converged"] == 1 and l1(x, Xn) <= 1e-14


def test_per_sweep_pins():
    """SURVEY App. B per-sweep pins: bulk DI-CYC on the chain gives H=[.075,.075] then
    [.075,.13875]; sequential DI-CYC on spec3 converges in one cycle via the loop fold."""
    src, dst = links_arrays([(0, 1)])
    F = np.full(2, 0.075)
    H = np.zeros(2)
    s1 = oracle.bulk_sweep(src, dst, 2, F, H, 0.0, r=F.sum(), d=D, variant="cyc")
    assert np.array_equal(s1["H"], [0.075, 0.075])
    s2 = oracle.bulk_sweep(src, dst, 2, s1["F"], s1["H"], s1["e"], r=s1["F"].sum(), d=D, variant="cyc")
    assert np.allclose(s2["H"], [0.075, 0.13875], rtol=0, atol=1e-16)   # a few ulps
    assert s2["F"].sum() == 0.0
    src, dst = links_arrays([(0, 1), (1, 2), (2, 2)])
    H, F, st = oracle.di(src, dst, 3, d=D, tol=1e-16, variant="cyc")
    assert st["cycles"] == 1 and F.sum() == 0.0
    assert abs(H[2] - 0.8575) <= 1e-15
    # bulk DI-CYC needs 3 sweeps (depth-2 chain)
    H, F, st = oracle.bulk_di(src, dst, 3, d=D, tol=1e-16, variant="cyc")
    assert st["cycles"] == 3


# ------------------------------------------------------------ starvation guard
@pytest.mark.parametrize("links,n", [([(0, 1)], 2), ([(0, 1), (1, 2), (2, 0)], 3), ([(0, 0)], 1)],
                         ids=["chain", "cycle3", "selfloop"])
def test_starvation_guard(links, n):
    """Strict '>' starves on these graphs (reading G5); the guard keeps progress."""
    src, dst = links_arrays(links)
    X = defn.solve_dense(src, dst, n, D)
    H, F, st = oracle.di(src, dst, n, d=D, tol=1e-15, variant="sop")
    assert st["converged"] == 1 and st["guard_sweeps"] > 0
    assert l1(H, X) <= 1e-13


# ----------------------------------------------------- random graphs vs dense solve
CORPUS = [digen.small_random(s) for s in range(200)]


@pytest.mark.parametrize("d", [0.5, 0.85, 0.95])
def test_random_vs_dense(d):
    """T2: every oracle solver vs numpy.linalg.solve on 200 random graphs (loops, dups, dangling)."""
    for k, (src, dst, n) in enumerate(CORPUS):
        X = defn.solve_dense(src, dst, n, d)
        Xn = X / X.sum()
        for variant in ("cyc", "sop"):
            H, F, st = oracle.di(src, dst, n, d=d, tol=1e-15, variant=variant)
            assert st["converged"] == 1
            assert l1(H, X) <= 1e-13, (k, variant)
            H, F, st = oracle.bulk_di(src, dst, n, d=d, tol=1e-15, variant=variant)
            assert l1(H, X) <= 1e-13, (k, "bulk", variant)
        x, st = oracle.gs(src, dst, n, d=d, target=1e-15)
        assert l1(x, X) <= 1e-13, (k, "gs")
        x1, st1, h1 = oracle.pi(src, dst, n, d=d, target=1e-15, history=True)
        x2, st2, h2 = oracle.pi_col(src, dst, n, d=d, target=1e-15, history=True)
        assert l1(x1, Xn) <= 1e-13 and l1(x2, Xn) <= 1e-13, (k, "pi")


def test_pi_lockstep():
    """PI and PI' compute the same iterate: equal sweep counts at target 1e-10 and
    per-sweep error estimates within 1e-12; the paper's equal 'nb iter' columns."""
    for k, (src, dst, n) in enumerate(CORPUS):
        x1, st1, h1 = oracle.pi(src, dst, n, d=D, target=1e-10, history=True)
        x2, st2, h2 = oracle.pi_col(src, dst, n, d=D, target=1e-10, history=True)
        assert st1["cycles"] == st2["cycles"], k
        assert np.max(np.abs(h1 - h2)) <= 1e-12 and np.max(np.abs(x1 - x2)) <= 1e-12


def test_invariants_mid_run():
    """F = B + P.H - H elementwise, conservation, error bound and H <= X at arbitrary stops."""
    for k, (src, dst, n) in enumerate(CORPUS[:80]):
        X = defn.solve_dense(src, dst, n, D)
        P = defn.dense_P(src, dst, n, D)
        B = defn.uniform_B(n, D)
        out = np.bincount(src, minlength=n)
        for variant in ("cyc", "sop"):
            for cycles in (1, 2, 5):
                H, F, st = oracle.di(src, dst, n, d=D, tol=1e-300, variant=variant, max_cycles=cycles)
                assert np.all(F >= 0)
                assert np.abs(F - (B + P @ H - H)).max() <= 1e-15, (k, variant, cycles)
                cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
                assert abs(cons - (1 - D)) <= 1e-14
                assert l1(X, H) <= F.sum() / (1 - D) + 1e-15
                assert np.all(H <= X + 1e-15)


def test_bulk_q_plus_s_predicts_r():
    """r_{n+1} = q_n + s_n for the bulk sweep."""
    for src, dst, n in CORPUS[:60]:
        F = defn.uniform_B(n, D)
        H = np.zeros(n)
        e = 0.0
        for _ in range(6):
            r = F.sum()
            res = oracle.bulk_sweep(src, dst, n, F, H, e, r=r, d=D, variant="sop")
            assert abs(res["F"].sum() - (res["q"] + res["s"])) <= 1e-15
            F, H, e = res["F"], res["H"], res["e"]


def test_bulk_cyc_neumann():
    """Bulk DI-CYC without self-loops: F_n = P^n B and H_n = sum_{k<n} P^k B (closed form)."""
    src, dst, n = digen.make("c1")
    P = defn.sparse_P(src, dst, n, D)
    B = defn.uniform_B(n, D)
    F, H, e = B.copy(), np.zeros(n), 0.0
    Fn, Hn = B.copy(), np.zeros(n)
    for _ in range(10):
        res = oracle.bulk_sweep(src, dst, n, F, H, e, r=F.sum(), d=D, variant="cyc")
        F, H, e = res["F"], res["H"], res["e"]
        Hn = Hn + Fn
        Fn = P @ Fn
        nz = Fn > 0
        assert np.array_equal(F > 0, nz)
        assert np.max(np.abs(F[nz] - Fn[nz]) / Fn[nz]) <= 1e-13
        assert np.max(np.abs(H - Hn) / np.maximum(Hn, 1e-300)) <= 1e-13


def test_closure_drainage():
    """Nodes of the recursive zero in-degree set E at depth <= t hold exactly 0.0 fluid after
    t+1 bulk DI-CYC sweeps (P:132-135 'converged exactly in finite steps')."""
    for seed in range(100):
        src, dst, n = digen.dag_fringe(seed)
        depth = digen.closure(src, dst, n)
        F, H, e = defn.uniform_B(n, D), np.zeros(n), 0.0
        for t in range(8):
            res = oracle.bulk_sweep(src, dst, n, F, H, e, r=F.sum(), d=D, variant="cyc")
            F, H, e = res["F"], res["H"], res["e"]
            drained = (depth >= 0) & (depth <= t)
            assert np.all(F[drained] == 0.0), (seed, t)


def test_closure_brute_force():
    """digen.closure matches a brute-force least fixpoint on random graphs."""
    for seed in range(100):
        src, dst, n = digen.small_random(seed, n_max=30)
        inn = [set() for _ in range(n)]
        for s, t in zip(src.tolist(), dst.tolist()):
            inn[t].add(s)
        E = set()
        changed = True
        while changed:
            changed = False
            for j in range(n):
                if j not in E and j not in inn[j] and inn[j] <= E:
                    E.add(j)
                    changed = True
        depth = digen.closure(src, dst, n)
        assert set(np.nonzero(depth >= 0)[0].tolist()) == E


def test_c1_vs_spsolve():
    """T3: oracle DI (both variants) vs scipy spsolve at C1 seeds 1-3."""
    for seed in (1, 2, 3):
        src, dst, n = digen.make("c1", seed=seed)
        X = defn.solve_sparse(src, dst, n, D)
        for variant in ("sop", "cyc"):
            H, F, st = oracle.di(src, dst, n, d=D, tol=1e-13, variant=variant)
            assert st["converged"] == 1 and l1(H, X) <= 1e-12


def test_paper_stop_mode():
    """Paper stop: sum F/(1-d-d e) <= 1/N. It must stop no later than the raw 1e-10 stop,
    and the normalised estimate upper-bounds the true normalised error within a factor 2."""
    src, dst, n = digen.make("c1")
    X = defn.solve_sparse(src, dst, n, D)
    H, F, st = oracle.di(src, dst, n, d=D, tol=1.0 / n, variant="sop", paper_stop=True)
    assert st["converged"] == 1
    err = st["residual"] / (1 - D - D * st["e"])
    assert err <= 1.0 / n
    assert l1(H / H.sum(), X / X.sum()) <= 2 * err


def test_invalid_args():
    src, dst = links_arrays([(0, 1)])
    with pytest.raises(ValueError):
        oracle.di(src, dst, 2, d=1.0)
    with pytest.raises(ValueError):
        oracle.di(src, np.array([5], dtype=np.int32), 2)
