"""Experiment: DI-SOP threshold scale alpha (F4) on the asynchronous cycle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
for alpha in [float(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "0.5,1,1.5,2,3,4").split(",")]:
    g.set_threshold_scale(alpha)
    g.solve(d=0.85, tol=1e-10, asynchronous=True)
    sts = [g.solve(d=0.85, tol=1e-10, asynchronous=True) for _ in range(2)]
    st = min(sts, key=lambda s: s["solve_ms"])
    print(cfg, "alpha", alpha, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"], "eq",
          round(st["equivalent_iterations"], 2), "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1), flush=True)
