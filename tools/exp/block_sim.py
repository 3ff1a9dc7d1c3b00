"""CPU simulation (numpy/scipy, experiment only): link diffusions to ||F||_1 <= tol for the
block-ordered bulk DI-SOP (K ordered node blocks per cycle, r fixed per cycle as in P:294-298)
and a threshold scale alpha. No self-loops (configs drop them)."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, scipy.sparse as sp
import digen

def run(src, dst, n, K=1, alpha=1.0, d=0.85, tol=1e-10, r_per_block=False, order=None):
    L = len(src)
    out = np.bincount(src, minlength=n).astype(np.float64)
    A = sp.csc_matrix((np.ones(L), (dst, src)), shape=(n, n))   # column i = out-links of i
    F = np.full(n, (1 - d) / n); H = np.zeros(n)
    bounds = np.linspace(0, n, K + 1).astype(np.int64)
    links = 0; cycles = 0
    while F.sum() > tol and cycles < 5000:
        r = F.sum(); t = r / L * alpha
        for b in range(K):
            lo, hi = bounds[b], bounds[b + 1]
            if r_per_block:
                t = F.sum() / L * alpha
            f = F[lo:hi]; o = out[lo:hi]
            sel = f > t * o
            if not sel.any():
                continue
            T = np.where(sel, f, 0.0)
            H[lo:hi] += T; F[lo:hi] = np.where(sel, 0.0, f)
            nd = sel & (o > 0)
            v = np.zeros(n); v[lo:hi][nd] = T[nd] * d / o[nd]
            links += int(o[nd].sum())
            F += A @ v
        cycles += 1
    return links / L, cycles

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
src, dst, n = digen.make(cfg, n=n_override) if n_override else digen.make(cfg)
print(cfg, n, len(src), flush=True)
for K in ([1, 8, 16] if len(sys.argv) > 3 else [1, 2, 4, 8, 16, 64]):
    t0 = time.time()
    eq, cyc = run(src, dst, n, K=K)
    print(f"K={K:3d} alpha=1   eq_iter={eq:.2f} cycles={cyc} ({time.time()-t0:.0f}s)", flush=True)
for a in ([] if len(sys.argv) > 3 else [1.5, 2.0]):
    eq, cyc = run(src, dst, n, K=1, alpha=a)
    print(f"K=  1 alpha={a} eq_iter={eq:.2f} cycles={cyc}", flush=True)

if len(sys.argv) > 3 and sys.argv[3] == "orders":
    indeg = np.bincount(dst, minlength=n)
    rank = np.argsort(-indeg, kind="stable")           # rank r -> old id
    P = 4096; M = n // P
    r = np.arange(n); new = (r % P) * M + (r // P)     # striped (n divisible by P here)
    new_of = np.empty(n, np.int64); new_of[rank] = new
    s2, t2 = new_of[src], new_of[dst]
    for K in [1, 8, 16, 32]:
        eq, cyc = run(s2, t2, n, K=K)
        print(f"striped-indeg K={K:3d} eq_iter={eq:.2f} cycles={cyc}", flush=True)
    new_of2 = np.empty(n, np.int64); new_of2[rank] = np.arange(n)
    for K in [8, 16]:
        eq, cyc = run(new_of2[src], new_of2[dst], n, K=K)
        print(f"plain-indeg K={K:3d} eq_iter={eq:.2f} cycles={cyc}", flush=True)
