"""oracle.definition — the result the method reaches, written as its plain definition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §1: X = P.X + B. With the PageRank instantiation of §2.5
(P:166): P_ji = d/#out_i for every link i->j (a link listed twice counts
twice; a self-loop i->i contributes P_ii), dangling columns are zero, B = (1-d)/N.
Since every column sum of P is <= d < 1, I - P is invertible and X is unique; the
oracle for the converged history H is therefore X = (I - P)^{-1} B, computed with a
library linear solve (numpy dense LU for small N, scipy sparse LU for larger N).
"""
from __future__ import annotations

import numpy as np


def dense_P(src, dst, n, d):
    """Dense P (n x n, fp64): P[j, i] += d / out_i for every link i -> j."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    out = np.bincount(src, minlength=n).astype(np.float64)
    P = np.zeros((n, n), dtype=np.float64)
    np.add.at(P, (dst, src), d / out[src])
    return P


def sparse_P(src, dst, n, d):
    import scipy.sparse as sp
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    out = np.bincount(src, minlength=n).astype(np.float64)
    vals = d / out[src] if len(src) else np.zeros(0)
    return sp.csr_matrix((vals, (dst, src)), shape=(n, n))   # duplicates are summed


def uniform_B(n, d):
    return np.full(n, (1.0 - d) / n, dtype=np.float64)


def solve_dense(src, dst, n, d, B=None):
    """X = (I - P)^{-1} B by numpy.linalg.solve (n small)."""
    B = uniform_B(n, d) if B is None else np.asarray(B, dtype=np.float64)
    return np.linalg.solve(np.eye(n) - dense_P(src, dst, n, d), B)


def solve_sparse(src, dst, n, d, B=None):
    """X = (I - P)^{-1} B by scipy.sparse.linalg.spsolve (sparse LU)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    B = uniform_B(n, d) if B is None else np.asarray(B, dtype=np.float64)
    A = (sp.identity(n, format="csc") - sparse_P(src, dst, n, d).tocsc()).tocsc()
    return spl.spsolve(A, B)


def solve_exact(links, n, d):
    """Exact rational X = (I - P)^{-1} B (Fractions, Gauss-Jordan); d must be a Fraction.
    For the tiny hand-checkable pins of tests/golden/pins.txt."""
    from fractions import Fraction
    out = [0] * n
    for s, _ in links:
        out[s] += 1
    M = [[Fraction(int(i == j)) for j in range(n)] + [(1 - d) / n] for i in range(n)]
    for s, t in links:
        M[t][s] -= d / out[s]
    for c in range(n):
        p = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    return [M[i][n] / M[i][i] for i in range(n)]
