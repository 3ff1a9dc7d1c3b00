"""T5: device CSR/CSC builder vs a numpy lexsort reference, byte for byte."""
import numpy as np
import pytest

import digen
from gpu_util import csr_reference, need_gpu, upload, warm_count, warm_shift

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dedup,drop_self", [(False, False), (True, False), (False, True), (True, True)])
def test_builder_random(dedup, drop_self):
    need_gpu()
    for seed in range(40):
        src, dst, n = digen.small_random(seed, n_max=300)
        g = upload(src, dst, n, dedup=dedup, drop_self_loops=drop_self, build_csc=True, reorder=False)
        ref = csr_reference(src, dst, n, dedup, drop_self)
        got = g.test_csr(csc=True)
        assert g.n_links == len(ref["col"])
        for k in ("row_ptr", "col", "deg", "kloop"):
            assert np.array_equal(got[k], ref[k]), (seed, k)
        # CSC = CSR of the reversed kept links
        rc = csr_reference(ref["dst"], ref["src"], n)
        assert np.array_equal(got["csc_ptr"], rc["row_ptr"]) and np.array_equal(got["csc_row"], rc["col"])
        g.free()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_builder_configs(name):
    need_gpu()
    src, dst, n = digen.make(name)
    perm = np.random.default_rng(0).permutation(len(src))   # builder must not rely on input order
    g = upload(src[perm], dst[perm], n, build_csc=True, reorder=False)
    got = g.test_csr(csc=True)
    ref = csr_reference(src, dst, n)
    for k in ("row_ptr", "col", "deg", "kloop"):
        assert np.array_equal(got[k], ref[k]), k
    g.free()


def test_builder_host_pointers_and_edges():
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.small_random(3, n_max=50)
    g = di.Graph(src, dst, n, reorder=False)      # host arrays -> DI_HOST_PTRS path
    ref = csr_reference(src, dst, n)
    assert np.array_equal(g.test_csr()["col"], ref["col"])
    g.free()
    g = di.Graph(np.zeros(0, np.int32), np.zeros(0, np.int32), 7)   # no links: all dangling
    c = g.test_csr()
    assert np.array_equal(c["row_ptr"], np.zeros(8)) and np.all(c["deg"] == 0)
    g.free()
    with pytest.raises(di.DIError) as ei:
        di.Graph(np.array([0, 5], np.int32), np.array([1, 1], np.int32), 3)
    assert ei.value.status == di.DI_EINVAL and "link 1" in str(ei.value)


@pytest.mark.parametrize("name,warm", [("c1", -1), ("c2", -1), ("c2", 4032), ("c2", 1000)])
def test_reorder_relabelling(name, warm):
    """Default upload relabels nodes by descending in-degree (stable): the internal CSR equals the
    reference CSR of the relabelled link list, byte for byte."""
    need_gpu()
    import paper_1204_6255_b200 as di
    src, dst, n = digen.make(name)
    with di.option("warm", warm):
        g = upload(src, dst, n, build_csc=True)
    old_of = g.test_perm()
    indeg = np.bincount(dst, minlength=n)
    ranked = np.argsort(-indeg, kind="stable")           # rank r -> caller id
    # placement (graph_build.cu k_place): on a skewed graph (top in-degree > 0.05 % of the links, kReplShare)
    # the 64 hottest ranks come first; when the first 4096 ranks take >= 10 % of the links and
    # n >= 8 * (W + hot), the next W ranks (warm tier, option warm: auto = 4032 on a B200, what
    # k_cycle's shared memory holds) go one every S ids after them (S = 2^s, the largest with
    # 8 * W * S <= n - hot); the rest in P stripes over the remaining ids in order,
    # P = largest prime <= (n - hot - W)/1024
    skewed = indeg.max() > 0.0005 * len(src) and n > 256
    hot = 64 if skewed else 0
    W = warm_count(indeg, len(src), n, warm, hot=hot)
    S = 1 << warm_shift(W, n - hot)

    def prime_at_most(x):
        if x < 2:
            return 1
        for p in range(x, 1, -1):
            if all(p % d for d in range(2, int(p ** 0.5) + 1)):
                return p
        return 1

    m = n - hot - W
    P = prime_at_most(max(1, m >> 10))
    r = np.arange(m)
    M, rem = m // P, m % P
    s_ = r % P
    c = s_ * M + np.minimum(s_, rem) + r // P
    if W:
        kq = c // (S - 1)
        c = np.where(kq < W, c + kq + 1, c + W)
    k = np.concatenate([np.arange(hot), hot + np.arange(W) * S, hot + c])
    expect = np.empty(n, np.int64)
    expect[k] = ranked
    assert np.array_equal(old_of, expect.astype(np.int32))
    new_of = np.empty(n, np.int64)
    new_of[old_of] = np.arange(n)
    ref = csr_reference(new_of[src], new_of[dst], n)
    got = g.test_csr(csc=True)
    for k in ("row_ptr", "col", "deg", "kloop"):
        assert np.array_equal(got[k], ref[k]), k
    g.free()


@pytest.mark.parametrize("row_sort", [0, 1])
def test_builder_row_sort_option(row_sort):
    """The two one-GPU builders (option row_sort: 64-bit key radix sort, or counting sort by source
    + per-row sorts by size class) give the byte-identical CSR, with and without the relabelling:
    random graphs with loops and duplicates, C1/C2 in shuffled input order, and rows in every size
    class (<= 16, <= 256, <= 4096 and hub rows of more than 4096 links, several segments)."""
    need_gpu()
    import paper_1204_6255_b200 as di
    rng = np.random.default_rng(5)
    n = 40000
    hub_src = np.concatenate([np.full(9000, 7), np.full(5000, 11), np.full(3000, 19), np.full(300, 23)])
    hub_dst = np.concatenate([rng.choice(n, 9000, replace=False), rng.choice(n, 5000, replace=False),
                              rng.integers(0, n, 3000), rng.integers(0, n, 300)])
    graphs = [digen.small_random(s, n_max=300)[:3] for s in range(20)]
    graphs += [(np.concatenate([rng.integers(0, n, 200000), hub_src]).astype(np.int32),
                np.concatenate([rng.integers(0, n, 200000), hub_dst]).astype(np.int32), n)]
    for name in ("c1", "c2"):
        s_, t_, nn = digen.make(name)
        perm = rng.permutation(len(s_))
        graphs.append((s_[perm], t_[perm], nn))
    with di.option("row_sort", row_sort):
        for src, dst, nn in graphs:
            ref = csr_reference(src, dst, nn)
            for reorder in (False, True):
                g = upload(src, dst, nn, reorder=reorder)
                got = g.test_csr()
                if reorder:   # compare in the internal numbering: the relabelled reference
                    old_of = g.test_perm()
                    new_of = np.empty(nn, np.int64)
                    new_of[old_of] = np.arange(nn)
                    r2 = csr_reference(new_of[src], new_of[dst], nn)
                else:
                    r2 = ref
                for k in ("row_ptr", "col", "deg", "kloop"):
                    assert np.array_equal(got[k], r2[k]), (nn, reorder, k)
                g.free()


def test_pipelined_host_upload():
    """Host link lists of >= 2^22 links take the pipelined upload (graph_build.cu: targets copied
    first and validated / counted while the sources follow in 8 chunks, keys made and sorted per
    chunk, sorted chunks merged): the CSR, CSC and relabelling are byte-identical to the upload of
    the same list from device memory (one key sort), with and without dedup / self-loop removal;
    a bad id anywhere is reported at its (first) link index like the one-shot path."""
    need_gpu()
    import paper_1204_6255_b200 as di
    rng = np.random.default_rng(21)
    n = 1 << 20
    L = 5_000_003   # ragged chunks
    src = (rng.zipf(1.6, L) % n).astype(np.int32)
    dst = (rng.zipf(1.4, L) % n).astype(np.int32)
    src[:1000] = dst[:1000]                        # self-loops
    src[1000:3000], dst[1000:3000] = src[5000:7000], dst[5000:7000]   # duplicates
    for kw in ({}, {"dedup": True, "drop_self_loops": True}, {"build_csc": True}):
        gh = di.Graph(src, dst, n, **kw)            # host arrays: DI_HOST_PTRS
        gd = upload(src, dst, n, **kw)              # device tensors
        a, b = gh.test_csr(csc=kw.get("build_csc", False)), gd.test_csr(csc=kw.get("build_csc", False))
        for k in a:
            assert np.array_equal(a[k], b[k]), (kw, k)
        assert np.array_equal(gh.test_perm(), gd.test_perm())
        gh.free()
        gd.free()
    ref = csr_reference(src, dst, n)
    g = di.Graph(src, dst, n, reorder=False)
    got = g.test_csr()
    for k in ("row_ptr", "col", "deg", "kloop"):
        assert np.array_equal(got[k], ref[k]), k
    g.free()
    for bad in ((3_000_000, None), (4_500_001, 4_000_000)):
        s2, d2 = src.copy(), dst.copy()
        s2[bad[0]] = -1 if bad[1] else s2[bad[0]]
        if bad[1] is None:
            d2[bad[0]] = n
        else:
            d2[bad[1]] = n + 5
        first = bad[0] if bad[1] is None else bad[1]
        with pytest.raises(di.DIError) as ei:
            di.Graph(s2, d2, n)
        assert ei.value.status == di.DI_EINVAL and f"link {first} " in str(ei.value), str(ei.value)
