"""Experiment: block-ordered cycles on a config (solve time, cycles, eq-iter per K)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=True)
g.solve(d=0.85, tol=1e-10, mode="auto")
st = min((g.solve(d=0.85, tol=1e-10, mode="auto") for _ in range(2)), key=lambda s: s["solve_ms"])
print(cfg, "auto K=1", round(st["solve_ms"], 2), st["sweeps"], round(st["equivalent_iterations"], 2), flush=True)
for K in [int(k) for k in (sys.argv[2].split(",") if len(sys.argv) > 2 else "1,4,8,16,32,64".split(","))]:
    g.solve(d=0.85, tol=1e-10, blocks=K)
    sts = [g.solve(d=0.85, tol=1e-10, blocks=K, profile=p) for p in (False, False, True)]
    st = min(sts[:2], key=lambda s: s["solve_ms"])
    pr = sts[2]
    print(cfg, "push K=%d" % K, round(st["solve_ms"], 2), st["sweeps"], round(st["equivalent_iterations"], 2),
          "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1),
          "push_ms", round(pr["push_ms"], 1), "select_ms", round(pr["select_ms"], 1), flush=True)
