"""Experiment: asynchronous cycles with and without the in-degree relabelling (reorder)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c3").split(","):
    src, dst, n = digen.make(cfg)
    for reorder in (True, False):
        g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, reorder=reorder)
        g.solve(d=0.85, tol=1e-10, asynchronous=True)
        sts = [g.solve(d=0.85, tol=1e-10, asynchronous=True) for _ in range(3)]
        st = min(sts, key=lambda s: s["solve_ms"])
        print(cfg, "reorder", reorder, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"], "eq",
              round(st["equivalent_iterations"], 2), "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1), flush=True)
        g.free()
