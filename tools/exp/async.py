"""Experiment: asynchronous cycles (DI_ASYNC) vs block-ordered cycles; agreement of H."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
ref = None
for name, kw in [("async", dict(asynchronous=True)),
                 ("async-graph", dict(asynchronous=True, graph_loop=True)), ("async-cyc", dict(asynchronous=True, variant="cyc"))]:
    g.solve(d=0.85, tol=1e-10, **kw)
    sts = [g.solve(d=0.85, tol=1e-10, **kw) for _ in range(3)]
    st = min(sts, key=lambda s: s["solve_ms"])
    H = g.history()
    if ref is None:
        ref = H.clone()
    print(cfg, name, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"], "eq", round(st["equivalent_iterations"], 2),
          "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1), "resid", st["residual_l1"],
          "conv", st["converged"], "dH", float((H - ref).abs().sum()), flush=True)
