"""Soak of the partitioned paths on emulated ranks: repeated solves (synchronous cycles through
peer memory, F2 rings, dense fallback, send/recv) on one graph per rank, each checked for
convergence and against the first solve's H."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import assemble, run_local_group
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
src, dst, n = digen.make(cfg)
modes = [dict(asynchronous=True), dict(asynchronous=True, dist_async=True),
         dict(asynchronous=True, exchange="dense"), dict(asynchronous=True, p2p=False), dict()]


def fn(r, grp):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    out = []
    with torch.cuda.stream(s):
        g = di.Graph(src, dst, n, rank=r, world=G, group=grp, stream=s)
        for k in range(reps):
            for m in modes:
                st = g.solve(d=0.85, tol=1e-10, **m)
                assert st["converged"] == 1, (k, m, st)
                out.append(g.history().cpu().numpy())
        rng = (g.lo, g.hi)
        g.free()
    return rng, out


t = time.time()
res = run_local_group(G, fn, timeout=1200)
ranges = [r for r, _ in res]
Hs = [assemble([o[k] for _, o in res], ranges, n) for k in range(len(res[0][1]))]
worst = max(float(np.abs(H - Hs[0]).sum()) for H in Hs)
print(cfg, "G", G, len(Hs), "solves ok; max ||H_k - H_0||_1 =", worst, "(<= 2e-10/(1-d) = 1.33e-9)",
      "wall", round(time.time() - t, 1), "s", flush=True)
assert worst <= 2e-10 / 0.15
