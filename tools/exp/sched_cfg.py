"""Experiment: the three schedules (bulk push, block-ordered K = 8, asynchronous cycles) on one
config, graph loop on: time, sweeps/cycles, eq-iter."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c3").split(","):
    src, dst, n = digen.make(cfg)
    g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
    for name, kw in (("bulk", {}), ("block8", dict(blocks=8)), ("async", dict(asynchronous=True))):
        g.solve(d=0.85, tol=1e-10, graph_loop=True, **kw)
        st = min((g.solve(d=0.85, tol=1e-10, graph_loop=True, **kw) for _ in range(3)), key=lambda s: s["solve_ms"])
        print(cfg, __import__("paper_1204_6255_b200").get_option("hot_acc"), name, "ms", round(st["solve_ms"], 2), "sweeps", st["sweeps"],
              "eq", round(st["equivalent_iterations"], 2), flush=True)
    g.free()
