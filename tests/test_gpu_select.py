"""T6: the select/compact step (a3+a4) on frozen (F, r) snapshots is bit-exact against the oracle's
bulk sweep (ids, bins, v = T*d/out, H, F), and its fused reductions q, s, e match."""
import numpy as np
import pytest

import digen
import oracle
from gpu_util import frontier_reference, need_gpu, upload

pytestmark = pytest.mark.gpu
D = 0.85


def snapshots(src, dst, n, variant, sweeps=(0, 1, 2, 7)):
    """(F, H, e, r) states produced by the ORACLE's bulk sweeps (never by the GPU)."""
    F = np.full(n, (1 - D) / n)
    H = np.zeros(n)
    e = 0.0
    out = []
    for k in range(max(sweeps) + 1):
        r = F.sum()
        if k in sweeps:
            out.append((F.copy(), H.copy(), e, r))
        res = oracle.bulk_sweep(src, dst, n, F, H, e, r=r, d=D, variant=variant)
        F, H, e = res["F"], res["H"], res["e"]
    return out


def check_select(g, src, dst, n, F, H, e, r, variant, bins):
    ref = oracle.bulk_sweep(src, dst, n, F, H, e, r=r, d=D, variant=variant)
    got = g.test_select(F, H, r, d=D, variant=variant)
    deg = np.bincount(src, minlength=n)
    ids, vals, chunk, off = frontier_reference(ref, deg, D, bins)
    assert np.array_equal(got["bin_off"], off)
    assert np.array_equal(got["ids"], ids)
    assert np.array_equal(got["vals"].view(np.uint64), vals.view(np.uint64))     # bitwise
    assert np.array_equal(got["chunk"], chunk)
    assert np.array_equal(got["H"].view(np.uint64), ref["H"].view(np.uint64))   # H += T bitwise
    Fsel = F.copy()
    Fsel[ref["mask"]] = 0.0
    assert np.array_equal(got["F"].view(np.uint64), Fsel.view(np.uint64))
    assert got["selected"] == int(ref["mask"].sum())
    assert got["links"] == int(deg[ref["mask"]].sum())
    # sums of n non-negative terms in different orders: |error| <= 2 n eps sum (Higham 4.2)
    tol = (2 * n + 4) * np.finfo(np.float64).eps
    for k in ("q", "s"):
        assert abs(got[k] - ref[k]) <= tol * abs(ref[k]), k
    assert abs(got["e"] - (ref["e"] - e)) <= tol * abs(ref["e"] - e) + 1e-300


@pytest.mark.parametrize("variant", ["sop", "cyc"])
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_select_bitexact_configs(name, variant):
    need_gpu()
    import paper_1204_6255_b200 as di
    bins = di.bins()
    src, dst, n = digen.make(name)
    g = upload(src, dst, n)
    for F, H, e, r in snapshots(src, dst, n, variant):
        check_select(g, src, dst, n, F, H, e, r, variant, bins)
    g.free()


def test_select_bitexact_loops_dups():
    """Random graphs with self-loops (fold, P:259-263 / G6) and parallel links, kept as given."""
    need_gpu()
    import paper_1204_6255_b200 as di
    bins = di.bins()
    for seed in range(30):
        src, dst, n = digen.small_random(seed, n_max=200)
        g = upload(src, dst, n)
        for variant in ("sop", "cyc"):
            for F, H, e, r in snapshots(src, dst, n, variant, sweeps=(0, 1, 3)):
                check_select(g, src, dst, n, F, H, e, r, variant, bins)
        g.free()


def test_select_hub_chunks():
    """A hub with > kChunk links lands in bin C as one entry per chunk, chunk index ascending."""
    need_gpu()
    import paper_1204_6255_b200 as di
    bins = di.bins()
    n = 5000
    rng = np.random.default_rng(1)
    hub_t = rng.choice(np.arange(1, n), size=4500, replace=False)
    src = np.concatenate([np.zeros(4500, np.int32), rng.integers(1, n, 3000).astype(np.int32)])
    dst = np.concatenate([hub_t.astype(np.int32), rng.integers(0, n, 3000).astype(np.int32)])
    key = np.unique(src.astype(np.int64) * n + dst)
    src, dst = (key // n).astype(np.int32), (key % n).astype(np.int32)
    g = upload(src, dst, n)
    F = rng.random(n) * 1e-4
    H = rng.random(n) * 1e-5
    check_select(g, src, dst, n, F, H, 0.0, F.sum(), "cyc", bins)
    got = g.test_select(F, H, F.sum(), d=D, variant="cyc")
    c0, c1 = got["bin_off"][3], got["bin_off"][4]
    assert c1 - c0 >= (4500 + bins["chunk"] - 1) // bins["chunk"]
    g.free()
