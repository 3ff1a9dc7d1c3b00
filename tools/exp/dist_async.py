"""Experiment: F2 asynchronous multi-GPU cycles (DI_DIST_ASYNC: no collective between cycles,
meetings every 4 cycles) vs synchronous asynchronous cycles (one exchange + header allgather per
cycle), on emulated ranks sharing one GPU: link diffusions (eq-iter), cycles, meetings. Times
are NOT multi-GPU times (the ranks share one GPU); the algorithmic effect of the staleness is."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import run_local_group
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
src, dst, n = digen.make(cfg)
for G in Gs:
    for da in (False, True):
        def fn(r, grp):
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                g = di.Graph(src, dst, n, rank=r, world=G, group=grp, stream=s)
                st = g.solve(d=0.85, tol=1e-10, asynchronous=True, dist_async=da)
                g.free()
            return st
        t = time.time()
        res = run_local_group(G, fn)
        st = res[0]
        print(cfg, "G", G, "dist_async" if da else "sync-cycles", "cycles", st["sweeps"], "meetings",
              st["meetings"], "eq", round(st["equivalent_iterations"], 2), "resid", st["residual_l1"],
              "conv", st["converged"], "wall s", round(time.time() - t, 2), flush=True)
