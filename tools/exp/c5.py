"""C5 (R-MAT N = 2^27, L ~ 2.16e9) on ONE B200: generate, upload from host pointers, asynchronous
DI-SOP to ||F||_1 <= 1e-10, then the properties that hold at any size (the oracle would need ~20 min
of one core per solve here): exact residual, conservation, F >= 0, and the invariant
F_i = B_i + (P.H)_i - H_i on 2000 sampled nodes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
D = 0.85
t = time.time()
src, dst, n = digen.make("c5")
print("generated N =", n, "L =", len(src), "in", round(time.time() - t, 1), "s", flush=True)
t = time.time()
g = di.Graph(src, dst, n)          # host pointers (DI_HOST_PTRS): H2D + build inside
torch.cuda.synchronize()
print("upload (H2D + build)", round(time.time() - t, 2), "s; device memory free",
      round(torch.cuda.mem_get_info()[0] / 1e9, 1), "GB", flush=True)
for k in range(3):
    st = g.solve(d=D, tol=1e-10, asynchronous=True, graph_loop=(k > 0))
    print("solve", k, "graph_loop" if k else "host loop", "ms", round(st["solve_ms"], 1), "cycles", st["sweeps"],
          "eq-iter", round(st["equivalent_iterations"], 2), "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1),
          "residual", st["residual_l1"], "converged", st["converged"], flush=True)
H = g.history().cpu().numpy()
resid, F = g.residual(return_F=True)
F = F.cpu().numpy()
g.free()
out = np.bincount(src, minlength=n).astype(np.float64)
cons = F.sum() + (1 - D) * H[out > 0].sum() + H[out == 0].sum()
print("residual", resid, "F >= 0:", bool(np.all(F >= 0)), "H >= 0:", bool(np.all(H >= 0)),
      "conservation error", abs(cons - (1 - D)), flush=True)
rng = np.random.default_rng(0)
sample = np.sort(rng.choice(n, 2000, replace=False))
mask = np.isin(dst, sample)
ph = np.zeros(n)
np.add.at(ph, dst[mask], D * H[src[mask]] / out[src[mask]])
inv = (1 - D) / n + ph[sample] - H[sample]
print("sampled invariant max |F - (B + P.H - H)| over 2000 nodes:", float(np.max(np.abs(inv - F[sample]))), flush=True)
