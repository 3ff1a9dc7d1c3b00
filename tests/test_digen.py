"""Generators: determinism, shape targets of BASELINE.json configs, sorted/deduped output."""
import numpy as np
import pytest

import digen


def test_thread_count_independent():
    a = digen.rmat(5000, 40000, p_dangling=0.15, p_zero_in=0.05, seed=7, threads=1)
    b = digen.rmat(5000, 40000, p_dangling=0.15, p_zero_in=0.05, seed=7, threads=5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = digen.host_block(20000, seed=3, threads=1)
    e = digen.host_block(20000, seed=3, threads=3)
    assert np.array_equal(c[0], e[0]) and np.array_equal(c[1], e[1])


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_shape(name):
    src, dst, n = digen.make(name)
    key = src.astype(np.int64) * n + dst
    assert np.all(np.diff(key) > 0)                 # sorted by (src, dst), no duplicates
    assert not np.any(src == dst)                   # self-loops removed
    st = digen.stats(src, dst, n)
    target_l = {"c1": 80_000, "c2": 10_000_000}[name]
    assert abs(st["l"] - target_l) / target_l < 0.05
    assert abs(st["d_over_n"] - 0.15) < 0.01        # ~15 % dangling
    if name == "c1":
        assert abs(st["zero_in_over_n"] - 0.05) < 0.01
    else:
        depth = digen.closure(src, dst, n)
        assert depth.max() >= 3                     # recursive zero in-degree chains
        assert abs(st["zero_in_over_n"] - 0.03) < 0.005


def test_c3_shape_small():
    src, dst, n = digen.make("c3", n=1 << 18)
    st = digen.stats(src, dst, n)
    assert abs(st["d_over_n"] - 0.10) < 0.01
    assert 10.5 < st["l_over_n"] < 12.5


def test_raw_keeps_duplicates():
    s, d = digen.rmat(256, 20000, raw=True, repair=False)
    key = s.astype(np.int64) * 256 + d
    assert np.all(np.diff(key) >= 0) and len(np.unique(key)) < len(key)


def test_paper_axes_workloads():
    """F3 input plumbing: P^T reverses every link; the loop-heavy stand-in adds one self-loop on
    ~20 % of the nodes (only nodes that already have out-links, so no new dangling change)."""
    import digen
    src, dst, n = digen.make("c1", seed=1)
    ts, tt = digen.transpose(src, dst)
    assert np.array_equal(ts, dst) and np.array_equal(tt, src)
    ls, lt = digen.add_self_loops(src, dst, n, frac=0.2)
    st = digen.stats(ls, lt, n)
    assert 0.17 <= st["o_over_n"] <= 0.23
    assert np.array_equal(np.bincount(ls, minlength=n) > 0, np.bincount(src, minlength=n) > 0)
    assert len(ls) - len(src) == int(np.sum(ls == lt))
