"""Experiment: k_cycle grid size vs order (a smaller grid is a narrower window of tiles in flight,
closer to the paper's sequential cycle, with less parallelism). the cycle_grid_div option is read per
process, so each setting runs in its own process (see the loop in the gpurun command)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
for cfg in sys.argv[1].split(","):
    src, dst, n = digen.make(cfg)
    g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
    g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    sts = [g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True) for _ in range(5)]
    st = min(sts, key=lambda s: s["solve_ms"])
    print(cfg, "div", __import__("paper_1204_6255_b200").get_option("cycle_grid_div"), "ms", round(st["solve_ms"], 3), "cycles", st["sweeps"],
          "eq", round(st["equivalent_iterations"], 2), flush=True)
    g.free()
