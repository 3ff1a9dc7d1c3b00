"""paper_1204_6255_b200 — B200-native D-iteration (arXiv:1204.6255) hot path.

Thin Python binding over the C ABI of ``libdi.so`` (include/di.h): argument marshalling
only. Every step of the solve runs in the library's sm_100a kernels; there is no CPU
fallback, and importing this package without the built library raises ImportError.
torch is used only for device memory and streams.

    import torch, paper_1204_6255_b200 as di
    g = di.Graph(src, dst, n)                       # src/dst: int32 (cuda tensors or host arrays)
    st = g.solve(d=0.85, tol=1e-10, variant="sop")  # DI-SOP sweeps to ||F||_1 <= 1e-10
    H = g.history()                                 # raw X estimate (torch float64, cuda)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdi.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python tools/build.py` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants (include/di.h)
DI_OK, DI_NOT_CONVERGED = 0, 1
DI_EINVAL, DI_ENOMEM, DI_ECUDA, DI_ENCCL, DI_ESTATE = -1, -2, -3, -4, -5
VARIANTS = {"sop": 0, "cyc": 1, "pi": 2, "pi_pull": 2, "pi_push": 3, "pi_col": 3, "gs": 4, "gs_block": 4}
DEDUP, DROP_SELF_LOOPS, BUILD_CSC, HOST_PTRS, LOCAL_LINKS, NO_REORDER = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
PUSH, PULL, AUTO, RESUME, PAPER_ERROR, TRACE, PROFILE, GRAPH_LOOP = 0x0, 0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40
ASYNC = 0x100
XCHG_SPARSE, XCHG_DENSE, XCHG_NOP2P, DIST_ASYNC = 0x200, 0x400, 0x800, 0x1000


class Stats(ctypes.Structure):
    _fields_ = [
        ("sweeps", ctypes.c_int64), ("selected_total", ctypes.c_int64),
        ("link_diffusions", ctypes.c_int64), ("starvation_fallbacks", ctypes.c_int64),
        ("nodes_scanned", ctypes.c_int64), ("pull_sweeps", ctypes.c_int64),
        ("gpu_launches", ctypes.c_int64),
        ("residual_l1", ctypes.c_double), ("dangling_absorbed", ctypes.c_double),
        ("equivalent_iterations", ctypes.c_double), ("solve_ms", ctypes.c_double),
        ("counted_bytes", ctypes.c_double), ("push_bytes", ctypes.c_double),
        ("push_ms", ctypes.c_double), ("select_ms", ctypes.c_double),
        ("error_estimate", ctypes.c_double), ("push_launches", ctypes.c_int64),
        ("converged", ctypes.c_int32), ("variant", ctypes.c_int32),
        ("exchange_bytes", ctypes.c_double), ("exchange_entries", ctypes.c_int64),
        ("exchange_ms", ctypes.c_double), ("dense_exchanges", ctypes.c_int64),
        ("p2p_exchanges", ctypes.c_int64), ("meetings", ctypes.c_int64),
        ("exchange_cold", ctypes.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("group", ctypes.c_void_p), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


_vp, _i64, _u32, _dbl, _ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double, ctypes.c_int
_lib.di_graph_upload.restype = _ci
_lib.di_graph_upload.argtypes = [_vp, _vp, _i64, _i64, _u32, _vp, _vp, ctypes.POINTER(_vp)]
_lib.di_graph_set_stream.restype = _ci
_lib.di_graph_set_stream.argtypes = [_vp, _vp]
_lib.di_graph_range.restype = _ci
_lib.di_graph_range.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
_lib.di_graph_links.restype = _ci
_lib.di_graph_links.argtypes = [_vp, ctypes.POINTER(_i64)]
_lib.di_solve.restype = _ci
_lib.di_solve.argtypes = [_vp, _dbl, _vp, _dbl, _ci, _i64, _u32, ctypes.POINTER(Stats)]
_lib.di_residual.restype = _ci
_lib.di_residual.argtypes = [_vp, ctypes.POINTER(_dbl), _vp]
_lib.di_history.restype = _ci
_lib.di_history.argtypes = [_vp, _vp]
_lib.di_sweep_log.restype = _ci
_lib.di_sweep_log.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, ctypes.POINTER(_i64)]
_lib.di_graph_free.restype = _ci
_lib.di_graph_free.argtypes = [_vp]
_lib.di_last_error.restype = ctypes.c_char_p
_lib.di_last_error.argtypes = []
_lib.di_set_option.restype = _ci
_lib.di_set_option.argtypes = [ctypes.c_char_p, _dbl]
_lib.di_get_option.restype = _ci
_lib.di_get_option.argtypes = [ctypes.c_char_p, ctypes.POINTER(_dbl)]
_lib.di_set_threshold_scale.restype = _ci
_lib.di_set_threshold_scale.argtypes = [_vp, _dbl]
_lib.di_nccl_unique_id.restype = _ci
_lib.di_nccl_unique_id.argtypes = [_vp]
_lib.di_group_create.restype = _ci
_lib.di_group_create.argtypes = [ctypes.c_int32, ctypes.POINTER(_vp)]
_lib.di_group_abort.restype = _ci
_lib.di_group_abort.argtypes = [_vp]
_lib.di_group_free.restype = _ci
_lib.di_group_free.argtypes = [_vp]
_lib.di_test_select.restype = _ci
_lib.di_test_select.argtypes = [_vp, _vp, _vp, _dbl, _dbl, _ci, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
_lib.di_test_cycle.restype = _ci
_lib.di_test_cycle.argtypes = [_vp, _vp, _vp, _dbl, _dbl, _ci, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.di_test_csr.restype = _ci
_lib.di_test_csr.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.di_test_perm.restype = _ci
_lib.di_test_perm.argtypes = [_vp, _vp]
_lib.di_test_bins.restype = _ci
_lib.di_test_bins.argtypes = [_vp]

EXPORTED = ["di_graph_upload", "di_graph_set_stream", "di_graph_range", "di_graph_links", "di_solve", "di_residual",
            "di_history", "di_sweep_log", "di_graph_free", "di_last_error",
            "di_nccl_unique_id", "di_group_create", "di_group_free", "di_group_abort",
            "di_set_threshold_scale", "di_set_option", "di_get_option",
            "di_test_select", "di_test_cycle", "di_test_csr", "di_test_bins", "di_test_perm"]


class DIError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libdi status {status}: {msg}")
        self.status = status


def _check(status, allow=(DI_OK,)):
    if status not in allow:
        raise DIError(status, _lib.di_last_error().decode(errors="replace"))
    return status


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def set_option(name: str, value) -> None:
    """di_set_option: process-wide tuning/diagnostic option (include/di.h lists them)."""
    _check(_lib.di_set_option(name.encode(), float(value)))


def get_option(name: str) -> float:
    v = _dbl()
    _check(_lib.di_get_option(name.encode(), ctypes.byref(v)))
    return v.value


class option:
    """Context manager: `with di.option("cold_bins", 1): ...` sets an option and restores it."""

    def __init__(self, name, value):
        self.name, self.value = name, value

    def __enter__(self):
        self.prev = get_option(self.name)
        set_option(self.name, self.value)
        return self

    def __exit__(self, *a):
        set_option(self.name, self.prev)


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (di_nccl_unique_id); create on one rank, broadcast the bytes."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.di_nccl_unique_id(buf))
    return buf.raw


class LocalGroup:
    """In-process group of `world` emulated ranks on one GPU (di_group): one host thread per rank,
    each building its own Graph(..., rank=r, group=this) and calling solve() concurrently."""

    def __init__(self, world):
        h = _vp()
        _check(_lib.di_group_create(int(world), ctypes.byref(h)))
        self._h = h
        self.world = int(world)

    def abort(self):
        """Wake every rank blocked in a group collective (they fail with DI_ESTATE)."""
        if getattr(self, "_h", None):
            _check(_lib.di_group_abort(self._h))

    def free(self):
        if getattr(self, "_h", None):
            _check(_lib.di_group_free(self._h))
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Graph:
    """Device graph handle (di_graph). src/dst: link list i -> j as int32, either CUDA tensors
    (device pointers) or host arrays / CPU tensors (copied with DI_HOST_PTRS).

    Partitioned: pass rank/world and either nccl_id (bytes from nccl_unique_id(),
    one process per GPU) or group (a LocalGroup, one thread per emulated rank). Every rank passes
    the full link list and owns the node range self.range() — or, with local_range=(lo, hi),
    only the links whose source lies in its own range [lo, hi) (DI_LOCAL_LINKS; the ranges tile
    [0, n) in rank order); history()/residual(return_F) are that rank's slice, residual() and
    solve() are collective."""

    def __init__(self, src, dst, n, dedup=False, drop_self_loops=False, build_csc=False,
                 reorder=True, stream=None, rank=0, world=1, nccl_id=None, group=None,
                 local_range=None):
        torch = _torch()
        self.n = int(n)
        flags = (DEDUP if dedup else 0) | (DROP_SELF_LOOPS if drop_self_loops else 0) | \
                (BUILD_CSC if build_csc else 0) | (0 if reorder else NO_REORDER) | \
                (LOCAL_LINKS if local_range is not None else 0)
        keep = []
        if isinstance(src, torch.Tensor) and src.is_cuda:
            s = src.to(torch.int32).contiguous()
            t = dst.to(torch.int32).contiguous()
            keep = [s, t]
            ps, pt, m = s.data_ptr(), t.data_ptr(), s.numel()
            self.device = s.device
        else:
            if isinstance(src, torch.Tensor):
                s = src.to(torch.int32).contiguous()
                t = dst.to(torch.int32).contiguous()
                keep = [s, t]
                ps, pt, m = s.data_ptr(), t.data_ptr(), s.numel()
            else:
                s = np.ascontiguousarray(src, dtype=np.int32)
                t = np.ascontiguousarray(dst, dtype=np.int32)
                keep = [s, t]
                ps, pt, m = s.ctypes.data, t.ctypes.data, s.size
            flags |= HOST_PTRS
            self.device = torch.device("cuda", torch.cuda.current_device())
        if m == 0:
            ps = pt = None
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = _vp()
        dist = None
        self._group = group
        if int(world) > 1 or nccl_id is not None or group is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
            lo, hi = local_range if local_range is not None else (0, 0)
            dist = Dist(int(rank), int(world),
                        ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None,
                        group._h if group is not None else None, int(lo), int(hi))
        _check(_lib.di_graph_upload(ps, pt, m, self.n, flags, self.stream.cuda_stream,
                                    ctypes.byref(dist) if dist is not None else None, ctypes.byref(h)))
        del keep
        self._h = h
        lk = _i64()
        _check(_lib.di_graph_links(self._h, ctypes.byref(lk)))
        self.n_links = int(lk.value)
        self.lo, self.hi = self.range()
        self.n_local = self.hi - self.lo

    # -------------------------------------------------------------- solve
    def solve(self, d=0.85, tol=1e-10, variant="sop", max_sweeps=100_000, B=None, resume=False,
              paper_error=False, trace=False, profile=False, mode="push", graph_loop=False,
              blocks=1, asynchronous=False, exchange="auto", p2p=True, dist_async=False,
              raise_on_not_converged=False):
        """di_solve. Returns the di_stats dict (status under key 'status').
        blocks=K > 1: block-ordered cycles (K ordered node blocks per cycle, push only).
        exchange ("auto" | "sparse" | "dense"): remote-fluid exchange of a partitioned graph;
        p2p=False moves the sparse lists with send/recv instead of peer-memory stores;
        dist_async=True (with asynchronous=True on a partitioned graph): no collective between
        cycles, the ranks meet every 4 cycles (F2)."""
        torch = _torch()
        flags = (RESUME if resume else 0) | (PAPER_ERROR if paper_error else 0) | \
                (TRACE if trace else 0) | (PROFILE if profile else 0) | \
                (GRAPH_LOOP if graph_loop else 0) | {"push": PUSH, "pull": PULL, "auto": AUTO}[mode] | \
                ((int(blocks) & 0xFF) << 16) | (ASYNC if asynchronous else 0) | \
                {"auto": 0, "sparse": XCHG_SPARSE, "dense": XCHG_DENSE}[exchange] | \
                (0 if p2p else XCHG_NOP2P) | (DIST_ASYNC if dist_async else 0)
        bp = None
        if B is not None:
            Bt = B if isinstance(B, torch.Tensor) else torch.as_tensor(np.asarray(B))
            Bt = Bt.to(device=self.device, dtype=torch.float64).contiguous()
            self._B = Bt
            bp = Bt.data_ptr()
        st = Stats()
        allow = (DI_OK,) if raise_on_not_converged else (DI_OK, DI_NOT_CONVERGED)
        rc = _check(_lib.di_solve(self._h, float(d), bp, float(tol), VARIANTS[variant], int(max_sweeps),
                                  flags, ctypes.byref(st)), allow)
        out = st.as_dict()
        out["status"] = rc
        return out

    def history(self):
        torch = _torch()
        H = torch.empty(self.n_local, dtype=torch.float64, device=self.device)
        _check(_lib.di_history(self._h, H.data_ptr()))
        return H

    def residual(self, return_F=False):
        torch = _torch()
        l1 = _dbl()
        F = torch.empty(self.n_local, dtype=torch.float64, device=self.device) if return_F else None
        _check(_lib.di_residual(self._h, ctypes.byref(l1), F.data_ptr() if F is not None else None))
        return (l1.value, F) if return_F else l1.value

    def sweep_log(self, cap=1 << 16):
        r = np.empty(cap, dtype=np.float64)
        sel = np.empty(cap, dtype=np.int64)
        lk = np.empty(cap, dtype=np.int64)
        mode = np.empty(cap, dtype=np.uint8)
        n = _i64()
        _check(_lib.di_sweep_log(self._h, r.ctypes.data, sel.ctypes.data, lk.ctypes.data, mode.ctypes.data,
                                 cap, ctypes.byref(n)))
        k = n.value
        return dict(r=r[:k].copy(), selected=sel[:k].copy(), links=lk[:k].copy(), mode=mode[:k].copy())

    def set_threshold_scale(self, alpha):
        """DI-SOP threshold scale alpha (F_i > alpha * r/L * #out_i; 1 = the paper's rule)."""
        _check(_lib.di_set_threshold_scale(self._h, float(alpha)))

    def set_stream(self, stream):
        """di_graph_set_stream: later calls of this handle enqueue on `stream` (a torch stream)."""
        _check(_lib.di_graph_set_stream(self._h, stream.cuda_stream))
        self.stream = stream

    def range(self):
        lo, hi = _i64(), _i64()
        _check(_lib.di_graph_range(self._h, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    # -------------------------------------------------------------- test-only
    def test_csr(self, csc=False):
        n, lk = self.n, self.n_links
        row_ptr = np.empty(n + 1, dtype=np.int64)
        col = np.empty(lk, dtype=np.int32)
        deg = np.empty(n, dtype=np.int32)
        kloop = np.empty(n, dtype=np.int32)
        cp = np.empty(n + 1, dtype=np.int64) if csc else None
        cr = np.empty(lk, dtype=np.int32) if csc else None
        _check(_lib.di_test_csr(self._h, row_ptr.ctypes.data, col.ctypes.data if lk else None,
                                deg.ctypes.data, kloop.ctypes.data,
                                cp.ctypes.data if csc else None, cr.ctypes.data if (csc and lk) else None))
        out = dict(row_ptr=row_ptr, col=col, deg=deg, kloop=kloop)
        if csc:
            out.update(csc_ptr=cp, csc_row=cr)
        return out

    def test_perm(self):
        old_of = np.empty(self.n, dtype=np.int32)
        _check(_lib.di_test_perm(self._h, old_of.ctypes.data))
        return old_of

    def test_select(self, F, H, r, d=0.85, variant="sop"):
        F = np.ascontiguousarray(F, dtype=np.float64)
        H = np.ascontiguousarray(H, dtype=np.float64)
        cap = 2 * self.n + self.n_links // 16 + 16
        ids = np.empty(cap, dtype=np.int32)
        vals = np.empty(cap, dtype=np.float64)
        chunk = np.empty(cap, dtype=np.int32)
        off = np.empty(5, dtype=np.int64)
        scal = np.empty(3, dtype=np.float64)
        cnt = np.empty(2, dtype=np.int64)
        Fo = np.empty(self.n, dtype=np.float64)
        Ho = np.empty(self.n, dtype=np.float64)
        _check(_lib.di_test_select(self._h, F.ctypes.data, H.ctypes.data, float(r), float(d), VARIANTS[variant],
                                   ids.ctypes.data, vals.ctypes.data, chunk.ctypes.data, cap,
                                   off.ctypes.data, scal.ctypes.data, cnt.ctypes.data, Fo.ctypes.data,
                                   Ho.ctypes.data))
        m = int(off[4])
        return dict(ids=ids[:m].copy(), vals=vals[:m].copy(), chunk=chunk[:m].copy(), bin_off=off.copy(),
                    q=scal[0], s=scal[1], e=scal[2], selected=int(cnt[0]), links=int(cnt[1]), F=Fo, H=Ho)

    def test_cycle(self, F, H, r, d=0.85, variant="sop"):
        """di_test_cycle: one record-mode cycle of k_cycle on the snapshot (F, H) with threshold
        fluid r; returns T, v (0 where not selected), F, H after, q, s, e, selected, links."""
        F = np.ascontiguousarray(F, dtype=np.float64)
        H = np.ascontiguousarray(H, dtype=np.float64)
        T = np.empty(self.n, dtype=np.float64)
        v = np.empty(self.n, dtype=np.float64)
        Fo = np.empty(self.n, dtype=np.float64)
        Ho = np.empty(self.n, dtype=np.float64)
        scal = np.empty(3, dtype=np.float64)
        cnt = np.empty(2, dtype=np.int64)
        _check(_lib.di_test_cycle(self._h, F.ctypes.data, H.ctypes.data, float(r), float(d), VARIANTS[variant],
                                  T.ctypes.data, v.ctypes.data, scal.ctypes.data, cnt.ctypes.data,
                                  Fo.ctypes.data, Ho.ctypes.data))
        return dict(T=T, v=v, F=Fo, H=Ho, q=scal[0], s=scal[1], e=scal[2], selected=int(cnt[0]),
                    links=int(cnt[1]))

    def free(self):
        if getattr(self, "_h", None):
            _lib.di_graph_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def bins():
    out = np.empty(4, dtype=np.int32)
    _check(_lib.di_test_bins(out.ctypes.data))
    return dict(T=int(out[0]), G=int(out[1]), W=int(out[2]), chunk=int(out[3]))
