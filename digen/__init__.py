"""digen — seeded synthetic link-list generators shared by the oracle and the CUDA path.

Input plumbing only: nothing here computes any part of the D-iteration (no P, no
fluid, no history). Both sides of every parity test receive the arrays returned
here. The configurations mirror BASELINE.json ``configs`` (C1..C5); the recipes
are in DESIGN.md §"Input recipe" and stand in for the paper's missing datasets
(§2.6, §2.8).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdigen.so")
_SRC = os.path.join(_HERE, "gen.c")
_GPU_SO = os.path.join(_HERE, "libdigen_gpu.so")
_GPU_SRC = os.path.join(_HERE, "gen_gpu.cu")
_NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False) -> str:
    """Compile gen.c into libdigen.so (gcc, host code) and gen_gpu.cu into libdigen_gpu.so (nvcc,
    sm_100a; per-source-range generation for partitioned runs) when nvcc is present."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    if os.path.exists(_NVCC) and (force or not os.path.exists(_GPU_SO)
                                  or os.path.getmtime(_GPU_SO) < os.path.getmtime(_GPU_SRC)):
        tmp = _GPU_SO + f".tmp{os.getpid()}"
        subprocess.check_call([_NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                               "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _GPU_SRC])
        os.replace(tmp, _GPU_SO)
    return _SO


_gpu_lib = None


def _G():
    global _gpu_lib
    if _gpu_lib is None:
        build()
        if not os.path.exists(_GPU_SO):
            raise RuntimeError(f"{_GPU_SO} is missing (needs nvcc)")
        lib = ctypes.CDLL(_GPU_SO)
        vp, i64, dbl, u64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int
        lib.digen_rmat_range_gpu.restype = ci
        lib.digen_rmat_range_gpu.argtypes = [i64, i64, dbl, dbl, dbl, u64, dbl, dbl, dbl, ci, ci, i64, i64,
                                             vp, i64, ctypes.POINTER(i64), vp]
        _gpu_lib = lib
    return _gpu_lib


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64, dbl, u64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_int
        lib.digen_rmat.restype = vp
        lib.digen_rmat.argtypes = [i64, i64, dbl, dbl, dbl, u64, dbl, dbl, dbl, ci, ci, ci, ci]
        lib.digen_hostblock.restype = vp
        lib.digen_hostblock.argtypes = [i64, i64, i64, dbl, dbl, dbl, dbl, u64, ci, ci]
        lib.digen_len.restype = i64
        lib.digen_len.argtypes = [vp]
        lib.digen_raw.restype = i64
        lib.digen_raw.argtypes = [vp]
        lib.digen_copy.restype = None
        lib.digen_copy.argtypes = [vp, vp, vp]
        lib.digen_free.restype = None
        lib.digen_free.argtypes = [vp]
        _lib = lib
    return _lib


def _take(h):
    lib = _L()
    if not h:
        raise ValueError("digen: invalid generator arguments")
    try:
        n = lib.digen_len(h)
        src = np.empty(n, dtype=np.int32)
        dst = np.empty(n, dtype=np.int32)
        lib.digen_copy(h, src.ctypes.data, dst.ctypes.data)
    finally:
        lib.digen_free(h)
    return src, dst


def rmat(n: int, m: int, a: float = 0.57, b: float = 0.19, c: float = 0.19, seed: int = 1,
         p_dangling: float = 0.0, p_zero_in: float = 0.0, chain_heads: float = 0.0,
         repair: bool = True, repair_in: bool = True, raw: bool = False, threads: int = 0):
    """R-MAT + repair link list (sorted by (src,dst); deduped, no self-loops unless raw)."""
    h = _L().digen_rmat(n, m, a, b, c, seed, p_dangling, p_zero_in, chain_heads,
                        int(repair), int(repair_in), int(raw), threads)
    return _take(h)


def host_block(n: int, bmin: int = 64, bmax: int = 1024, p_dangling: float = 0.10,
               mean_out: float = 12.0 / 0.9, p_intra: float = 0.8, alpha_in: float = 2.1,
               seed: int = 1, raw: bool = False, threads: int = 0):
    """Host-block locality link list (BASELINE.json configs[2])."""
    h = _L().digen_hostblock(n, bmin, bmax, p_dangling, mean_out, p_intra, alpha_in, seed, int(raw), threads)
    return _take(h)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    kind: str
    params: dict
    note: str


# BASELINE.json configs[0..4]. M (R-MAT candidates) calibrated so L lands near the target.
CONFIGS = {
    "c1": Config("c1", 10_000, "rmat",
                 dict(m=104_000, a=0.57, b=0.19, c=0.19, p_dangling=0.15, p_zero_in=0.05),
                 "R-MAT(0.57,0.19,0.19,0.05) N=1e4 L~80k, 15% dangling, 5% zero-in"),
    "c2": Config("c2", 1_000_000, "rmat",
                 dict(m=11_100_000, a=0.55, b=0.10, c=0.25, p_dangling=0.17, p_zero_in=0.0,
                      chain_heads=0.03),
                 "asymmetric R-MAT N=1e6 L~10M, 15% dangling, zero-in chains at 3% of nodes"),
    "c3": Config("c3", 8_388_608, "hostblock",
                 dict(bmin=64, bmax=1024, p_dangling=0.10, mean_out=12.0 / 0.9, p_intra=0.8, alpha_in=2.1),
                 "host-block N=2^23, blocks U{64..1024}, 80% intra, avg out 12, 10% dangling"),
    "c4": Config("c4", 1 << 24, "rmat",
                 dict(m=int(17.5 * (1 << 24)), a=0.57, b=0.19, c=0.19, p_dangling=0.12, p_zero_in=0.0,
                      repair_in=False),
                 "R-MAT(0.57,0.19,0.19,0.05) N=2^24 L~268M, 12% dangling, natural zero-in"),
    "c5": Config("c5", 1 << 27, "rmat",
                 dict(m=int(17.5 * (1 << 27)), a=0.57, b=0.19, c=0.19, p_dangling=0.12, p_zero_in=0.0,
                      repair_in=False),
                 "R-MAT N=2^27 L~2.1B, 12% dangling"),
}


def make(name: str, seed: int = 1, n: int | None = None, threads: int = 0):
    """Generate config `name` (optionally at a reduced node count n, same recipe)."""
    cfg = CONFIGS[name]
    nn = cfg.n if n is None else int(n)
    p = dict(cfg.params)
    if cfg.kind == "rmat":
        m = p.pop("m")
        if n is not None:
            m = int(round(m * nn / cfg.n))
        src, dst = rmat(nn, m, seed=seed, threads=threads, **p)
    else:
        src, dst = host_block(nn, seed=seed, threads=threads, **p)
    return src, dst, nn


def node_ranges(n: int, world: int):
    """Equal node ranges [n*g/world, n*(g+1)/world) (the R-MAT + repair ids are Feistel-relabelled,
    so equal ranges carry about equal link counts)."""
    return [(n * g // world, n * (g + 1) // world) for g in range(world)]


def make_range_gpu(name: str, lo: int, hi: int, seed: int = 1, n: int | None = None, device=None):
    """The links of config `name` (an R-MAT config) whose source lies in [lo, hi), generated on the
    GPU: torch int32 CUDA tensors (src, dst) sorted by (src, dst), deduplicated, no self-loops —
    exactly `make(name)`'s links with a source in [lo, hi) (tests/test_gpu_digen.py), without
    drawing the rest of the graph on the host (C5 at G = 8: ~270M links per rank)."""
    import torch
    cfg = CONFIGS[name]
    if cfg.kind != "rmat":
        raise ValueError(f"make_range_gpu: {name} is not an R-MAT config")
    nn = cfg.n if n is None else int(n)
    p = dict(cfg.params)
    m = p.pop("m")
    if n is not None:
        m = int(round(m * nn / cfg.n))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    expect = (m + nn) * (hi - lo) / max(nn, 1)
    if expect > 1.0e9:   # torch.sort takes < 2^31 keys: sub-ranges, concatenated in order
        k = int(expect // 1.0e9) + 1
        parts = [make_range_gpu(name, lo + (hi - lo) * q // k, lo + (hi - lo) * (q + 1) // k, seed, n, dev)
                 for q in range(k)]
        return torch.cat([p_[0] for p_ in parts]), torch.cat([p_[1] for p_ in parts]), nn
    stream = torch.cuda.current_stream(dev)
    lib = _G()
    cap = int(1.15 * expect) + 4096
    for _ in range(3):
        keys = torch.empty(cap, dtype=torch.int64, device=dev)
        cnt = ctypes.c_int64(0)
        rc = lib.digen_rmat_range_gpu(nn, m, p.get("a", 0.57), p.get("b", 0.19), p.get("c", 0.19), seed,
                                      p.get("p_dangling", 0.0), p.get("p_zero_in", 0.0),
                                      p.get("chain_heads", 0.0), 1, int(p.get("repair_in", True)),
                                      int(lo), int(hi), keys.data_ptr(), cap, ctypes.byref(cnt),
                                      stream.cuda_stream)
        if rc != 0:
            raise RuntimeError(f"digen_rmat_range_gpu failed ({rc})")
        if cnt.value <= cap:
            break
        cap = int(cnt.value * 1.05) + 4096
    keys = keys[:cnt.value]
    keys, _ = torch.sort(keys)
    keys = torch.unique_consecutive(keys)
    src = (keys >> 32).to(torch.int32)
    dst = (keys & 0xFFFFFFFF).to(torch.int32)
    del keys
    keep = src != dst
    return src[keep].contiguous(), dst[keep].contiguous(), nn


def transpose(src: np.ndarray, dst: np.ndarray):
    """P^T workload of the paper's tables: every link reversed (input plumbing)."""
    return np.ascontiguousarray(dst, dtype=np.int32), np.ascontiguousarray(src, dtype=np.int32)


def add_self_loops(src: np.ndarray, dst: np.ndarray, n: int, frac: float = 0.2, seed: int = 1):
    """Loop-heavy stand-in (O/N ~ frac, as the uk-2007 prefixes' 11-24 %): one self-loop
    on a hash-chosen fraction of the nodes that already have out-links. Returns (src, dst) sorted."""
    outd = np.bincount(src, minlength=n)
    rng = np.random.default_rng(seed * 7919 + 17)
    cand = np.nonzero(outd > 0)[0]
    pick = cand[rng.random(cand.size) < frac * n / max(cand.size, 1)]
    s = np.concatenate([np.asarray(src, np.int64), pick])
    t = np.concatenate([np.asarray(dst, np.int64), pick])
    order = np.lexsort((t, s))
    return s[order].astype(np.int32), t[order].astype(np.int32)


def stats(src: np.ndarray, dst: np.ndarray, n: int) -> dict:
    """Table-1 style shape statistics (§2.4): L, D, zero-in, O, max_in, max_out.
    E (the recursive closure) is computed by closure_size()."""
    outd = np.bincount(src, minlength=n)
    ind = np.bincount(dst, minlength=n)
    return dict(n=int(n), l=int(len(src)), l_over_n=len(src) / n,
                d_over_n=float(np.mean(outd == 0)), zero_in_over_n=float(np.mean(ind == 0)),
                o_over_n=float(np.mean(np.bincount(src[src == dst], minlength=n) > 0)),
                max_in=int(ind.max(initial=0)), max_out=int(outd.max(initial=0)))


def closure(src: np.ndarray, dst: np.ndarray, n: int) -> np.ndarray:
    """Recursive zero in-degree set E with closure depth per node (-1 = not in E).
    Depth 0 = in-degree 0; else 1 + max depth over in-neighbours; self-loop nodes are never in E.
    Kahn-style peel over a CSR by destination (integer bookkeeping, not method arithmetic)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    remaining = np.bincount(dst, minlength=n).astype(np.int64)
    selfl = np.zeros(n, dtype=bool)
    selfl[src[src == dst]] = True
    order = np.argsort(src, kind="stable")
    s_sorted, d_sorted = src[order], dst[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=rp[1:])
    depth = np.full(n, -1, dtype=np.int64)
    frontier = np.nonzero((remaining == 0) & ~selfl)[0]
    depth[frontier] = 0
    level = 0
    while frontier.size:
        # out-links of the frontier
        starts, ends = rp[frontier], rp[frontier + 1]
        cnt = ends - starts
        if cnt.sum() == 0:
            break
        idx = np.repeat(starts - np.cumsum(np.concatenate(([0], cnt[:-1]))), cnt) + np.arange(cnt.sum())
        tg = d_sorted[idx]
        np.subtract.at(remaining, tg, 1)
        cand = np.unique(tg)
        newf = cand[(remaining[cand] == 0) & (depth[cand] < 0) & ~selfl[cand]]
        level += 1
        depth[newf] = level
        frontier = newf
    return depth


def small_random(seed: int, n_max: int = 64, loops: bool = True, dups: bool = True):
    """Small random link list for exhaustive tests (numpy PCG64, seeded): n in [1, n_max],
    up to 4n links, self-loops and parallel links allowed, dangling nodes left as drawn.
    Returned in random (unsorted) link order to exercise builders."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, n_max + 1))
    m = int(rng.integers(0, 4 * n + 1))
    src = rng.integers(0, n, size=m)
    dst = rng.integers(0, n, size=m)
    if not loops:
        keep = src != dst
        src, dst = src[keep], dst[keep]
    if dups and len(src):
        k = int(rng.integers(0, max(1, len(src) // 4) + 1))
        idx = rng.integers(0, len(src), size=k)
        src = np.concatenate([src, src[idx]])
        dst = np.concatenate([dst, dst[idx]])
        perm = rng.permutation(len(src))
        src, dst = src[perm], dst[perm]
    if not dups and len(src):
        key = np.unique(src.astype(np.int64) * n + dst)
        src, dst = key // n, key % n
        perm = rng.permutation(len(src))
        src, dst = src[perm], dst[perm]
    # make a fraction of nodes dangling on purpose
    if n > 2 and len(src):
        dang = rng.random(n) < 0.2
        keep = ~dang[src]
        src, dst = src[keep], dst[keep]
    return src.astype(np.int32), dst.astype(np.int32), n


def dag_fringe(seed: int, n: int = 40, depth: int = 6):
    """Random graph with a layered DAG fringe feeding a cyclic core (closure-drainage tests):
    layer 0 nodes have no in-links; layer k nodes receive links only from layers < k."""
    rng = np.random.default_rng(seed)
    layers = rng.integers(0, depth + 1, size=n)
    core = rng.random(n) < 0.3
    src, dst = [], []
    for j in range(n):
        if core[j]:
            for _ in range(int(rng.integers(1, 4))):
                src.append(int(rng.integers(0, n))); dst.append(j)
        elif layers[j] > 0:
            cands = np.nonzero((layers < layers[j]) & ~core)[0]
            if len(cands):
                for s in rng.choice(cands, size=min(len(cands), int(rng.integers(1, 4))), replace=False):
                    src.append(int(s)); dst.append(j)
    return np.array(src, dtype=np.int32), np.array(dst, dtype=np.int32), n
