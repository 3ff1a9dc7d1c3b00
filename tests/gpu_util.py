"""Shared helpers for the -m gpu tests (CPU references built from the oracle or numpy)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def upload(src, dst, n, **kw):
    import paper_1204_6255_b200 as di
    s = torch.from_numpy(np.ascontiguousarray(src, dtype=np.int32)).cuda()
    t = torch.from_numpy(np.ascontiguousarray(dst, dtype=np.int32)).cuda()
    return di.Graph(s, t, n, **kw)


def l1(a, b):
    return float(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)).sum())


def csr_reference(src, dst, n, dedup=False, drop_self=False):
    """numpy lexsort CSR (integer bookkeeping only) for the bit-exact builder test."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    order = np.lexsort((dst, src))
    s, t = src[order], dst[order]
    keep = np.ones(len(s), dtype=bool)
    if drop_self:
        keep &= s != t
    if dedup and len(s):
        dup = np.zeros(len(s), dtype=bool)
        dup[1:] = (s[1:] == s[:-1]) & (t[1:] == t[:-1])
        keep &= ~dup
    s, t = s[keep], t[keep]
    deg = np.bincount(s, minlength=n).astype(np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    kloop = np.bincount(s[s == t], minlength=n).astype(np.int32)
    return dict(row_ptr=row_ptr, col=t.astype(np.int32), deg=deg, kloop=kloop, src=s, dst=t)


def frontier_reference(res, deg, d, bins):
    """Expected frontier of the select step from an oracle bulk sweep result `res`
    (mask and T per node): bins by out-degree, ascending id, v = T*d/out."""
    mask = res["mask"] & (deg > 0)
    ids = np.nonzero(mask)[0]
    o = deg[ids].astype(np.int64)
    T = res["T"][ids]
    v = (T * d) / o.astype(np.float64)
    b = np.where(o <= bins["T"], 0, np.where(o <= bins["G"], 1, np.where(o <= bins["W"], 2, 3)))
    out_ids, out_v, out_c, off = [], [], [], [0]
    for k in range(4):
        sel = b == k
        if k < 3:
            out_ids.append(ids[sel]); out_v.append(v[sel]); out_c.append(np.zeros(sel.sum(), dtype=np.int32))
        else:
            nch = (o[sel] + bins["chunk"] - 1) // bins["chunk"]
            out_ids.append(np.repeat(ids[sel], nch)); out_v.append(np.repeat(v[sel], nch))
            out_c.append(np.concatenate([np.arange(c) for c in nch]).astype(np.int32) if len(nch) else
                         np.zeros(0, dtype=np.int32))
        off.append(off[-1] + len(out_ids[-1]))
    return (np.concatenate(out_ids).astype(np.int32), np.concatenate(out_v),
            np.concatenate(out_c), np.array(off, dtype=np.int64))


def warm_count(indeg, n_links, n, warm=-1, hot=0, grid=148 * 4):
    """Warm ranks the relabelling places (graph_build.cu, no cold bins): an explicit count `warm` > 0
    whenever n >= 8 * (warm + hot); auto (-1: 4032, what k_cycle's shared memory holds on a B200)
    when moreover the 64 + 4032 first ranks take >= 10 % of the links and the graph has
    >= 32 links per warm slot of k_cycle's grid (148 SMs x 4 CTAs); else 0."""
    w = 4032 if warm < 0 else warm
    if w <= 0 or n < 8 * (w + hot):
        return 0
    if warm > 0:
        return w
    k = min(n, 64 + w)
    top = np.sort(np.asarray(indeg))[::-1][:k].sum()
    return w if (top >= 0.10 * n_links and n_links >= 32 * grid * k) else 0


def warm_shift(W, region):
    """Spacing of the warm tier's ids (graph_build.cu, option warm_shift = 0): the largest s with
    8 * W * 2^s <= region (the warm ids span about the first eighth of the region)."""
    s = 0
    while W and ((W << (s + 1)) << 3) <= region:
        s += 1
    return s
