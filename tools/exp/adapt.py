"""Experiment: F4's alternating-frontier damping (DI_ADAPT) on bulk DI-SOP sweeps: sweeps,
eq-iter, time and the per-sweep link share with and without it (DI_ADAPT_PHI = target share)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c4").split(","):
    src, dst, n = digen.make(cfg)
    g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=True)
    for mode in ("push", "auto"):
        for adapt in (False, True):
            g.solve(d=0.85, tol=1e-10, mode=mode, adapt=adapt)
            sts = [g.solve(d=0.85, tol=1e-10, mode=mode, adapt=adapt, trace=True) for _ in range(2)]
            st = min(sts, key=lambda s: s["solve_ms"])
            share = g.sweep_log()["links"] / len(src)
            print(cfg, mode, "adapt" if adapt else "plain", "phi", os.environ.get("DI_ADAPT_PHI", "0.3"),
                  "ms", round(st["solve_ms"], 2), "sweeps", st["sweeps"], "eq", round(st["equivalent_iterations"], 2),
                  "share first 10:", np.round(share[:10], 2).tolist(), flush=True)
    g.free()
