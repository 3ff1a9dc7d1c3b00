"""oracle — plain CPU oracle for the D-iteration hot path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. The product package (paper_1204_6255_b200) never
imports it and shares no code with it.

Two layers (DESIGN.md §"Oracle"):
  * ``definition``: the fixed point X of X = P.X + B (§1) by a
    direct linear solve of (I - P) X = B (numpy dense / scipy sparse LU);
  * ``di_oracle.c``: the paper's five loops (§2.5) as written,
    single-threaded C, fp64, -ffp-contract=off; plus the bulk-synchronous sweep
    reading (R1) that the GPU reformulation follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdioracle.so")
_SRC = os.path.join(_HERE, "di_oracle.c")


def build(force: bool = False) -> str:
    """Compile di_oracle.c (gcc -O2 -ffp-contract=off; no -ffast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Stats(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int64), ("diffusions", ctypes.c_int64),
                ("guard_sweeps", ctypes.c_int64), ("selected", ctypes.c_int64),
                ("converged", ctypes.c_int64), ("residual", ctypes.c_double),
                ("e", ctypes.c_double), ("eq_iter", ctypes.c_double),
                ("solve_seconds", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        sp = ctypes.POINTER(Stats)
        lib.orc_di.restype = ci
        lib.orc_di.argtypes = [vp, vp, i64, i64, dbl, vp, dbl, ci, i64, ci, vp, vp, sp, vp, i64]
        lib.orc_bulk_sweep.restype = i64
        lib.orc_bulk_sweep.argtypes = [vp, vp, i64, i64, dbl, vp, vp, vp, ci, dbl, vp, vp, vp, vp, vp]
        lib.orc_bulk_di.restype = ci
        lib.orc_bulk_di.argtypes = [vp, vp, i64, i64, dbl, vp, dbl, ci, i64, vp, vp, sp]
        for f in (lib.orc_pi, lib.orc_pi_col, lib.orc_gs):
            f.restype = ci
            f.argtypes = [vp, vp, i64, i64, dbl, dbl, i64, vp, sp, vp, i64]
        _lib = lib
    return _lib


def _links(src, dst):
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    if src.shape != dst.shape:
        raise ValueError("src/dst length mismatch")
    return src, dst


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def di(src, dst, n, d=0.85, tol=1e-10, variant="sop", B=None, max_cycles=100_000,
       paper_stop=False, history=False):
    """Sequential DI-CYC / DI-SOP. Returns (H, F, stats[, r_history])."""
    src, dst = _links(src, dst)
    H = np.empty(n, dtype=np.float64)
    F = np.empty(n, dtype=np.float64)
    Bv = None if B is None else np.ascontiguousarray(B, dtype=np.float64)
    st = Stats()
    cap = max_cycles + 1 if history else 0
    hist = np.empty(cap, dtype=np.float64) if history else None
    rc = _L().orc_di(_ptr(src), _ptr(dst), len(src), n, d, _ptr(Bv), tol, int(variant == "sop"),
                     max_cycles, int(paper_stop), H.ctypes.data, F.ctypes.data, ctypes.byref(st),
                     _ptr(hist), cap)
    if rc < 0:
        raise ValueError("oracle: invalid arguments")
    out = (H, F, st.as_dict())
    if history:
        out = out + (hist[: min(st.cycles + 1, cap)].copy(),)
    return out


def bulk_sweep(src, dst, n, F, H, e, r, d=0.85, variant="sop"):
    """One bulk-synchronous sweep on snapshot F (R1). F, H updated in place (copies
    returned). Returns dict(F, H, e, T, mask, q, s, count, diffusions)."""
    src, dst = _links(src, dst)
    F = np.array(F, dtype=np.float64, copy=True)
    H = np.array(H, dtype=np.float64, copy=True)
    ev = ctypes.c_double(e)
    T = np.empty(n, dtype=np.float64)
    m = np.empty(n, dtype=np.uint8)
    q, s = ctypes.c_double(), ctypes.c_double()
    diff = ctypes.c_int64(0)
    c = _L().orc_bulk_sweep(_ptr(src), _ptr(dst), len(src), n, d, F.ctypes.data, H.ctypes.data,
                            ctypes.byref(ev), int(variant == "sop"), r, T.ctypes.data, m.ctypes.data,
                            ctypes.byref(q), ctypes.byref(s), ctypes.byref(diff))
    if c < 0:
        raise ValueError("oracle: invalid arguments")
    return dict(F=F, H=H, e=ev.value, T=T, mask=m.astype(bool), q=q.value, s=s.value, count=int(c),
                diffusions=int(diff.value))


def bulk_di(src, dst, n, d=0.85, tol=1e-10, variant="sop", B=None, max_cycles=100_000):
    """Bulk-synchronous D-iteration to ||F||_1 <= tol. Returns (H, F, stats)."""
    src, dst = _links(src, dst)
    H = np.empty(n, dtype=np.float64)
    F = np.empty(n, dtype=np.float64)
    Bv = None if B is None else np.ascontiguousarray(B, dtype=np.float64)
    st = Stats()
    rc = _L().orc_bulk_di(_ptr(src), _ptr(dst), len(src), n, d, _ptr(Bv), tol, int(variant == "sop"),
                          max_cycles, H.ctypes.data, F.ctypes.data, ctypes.byref(st))
    if rc < 0:
        raise ValueError("oracle: invalid arguments")
    return H, F, st.as_dict()


def _iter(fn, src, dst, n, d, target, max_iter, history):
    src, dst = _links(src, dst)
    x = np.empty(n, dtype=np.float64)
    st = Stats()
    cap = max_iter if history else 0
    hist = np.empty(cap, dtype=np.float64) if history else None
    rc = fn(_ptr(src), _ptr(dst), len(src), n, d, target, max_iter, x.ctypes.data, ctypes.byref(st),
            _ptr(hist), cap)
    if rc < 0:
        raise ValueError("oracle: invalid arguments")
    out = (x, st.as_dict())
    if history:
        out = out + (hist[: min(st.cycles, cap)].copy(),)
    return out


def pi(src, dst, n, d=0.85, target=None, max_iter=100_000, history=False):
    """PI, power iteration per row. Returns (x normalised, stats)."""
    return _iter(_L().orc_pi, src, dst, n, d, target if target else 1.0 / n, max_iter, history)


def pi_col(src, dst, n, d=0.85, target=None, max_iter=100_000, history=False):
    """PI', power iteration per column, stop rule of PI [G10]."""
    return _iter(_L().orc_pi_col, src, dst, n, d, target if target else 1.0 / n, max_iter, history)


def gs(src, dst, n, d=0.85, target=None, max_iter=100_000, history=False):
    """GS, cyclic Gauss-Seidel. Returns (x raw, stats)."""
    return _iter(_L().orc_gs, src, dst, n, d, target if target else 1.0 / n, max_iter, history)
