"""Experiment: the GPU comparators (PI pull, PI' push, block Gauss-Seidel) on one config: time,
iterations and the paper-error reached (tol on each scheme's own error)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=True)
for v in ("pi_pull", "pi_push", "gs"):
    g.solve(d=0.85, tol=1e-10 / n, variant=v, max_sweeps=300)
    st = g.solve(d=0.85, tol=1e-10 / n, variant=v, max_sweeps=300)
    print(cfg, v, "ms", round(st["solve_ms"], 2), "iterations", st["sweeps"], "error", st["error_estimate"],
          "converged", st["converged"], flush=True)
