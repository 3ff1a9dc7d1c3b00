"""Experiment: host-batched loop vs DI_GRAPH_LOOP (device while node), C4, K blocks."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
for K in [int(k) for k in (sys.argv[2] if len(sys.argv) > 2 else "1,8,16,32").split(",")]:
    for gl in (False, True):
        g.solve(d=0.85, tol=1e-10, blocks=K, graph_loop=gl)
        sts = [g.solve(d=0.85, tol=1e-10, blocks=K, graph_loop=gl) for _ in range(3)]
        st = min(sts, key=lambda s: s["solve_ms"])
        print(cfg, "K", K, "graph_loop", gl, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"],
              "eq", round(st["equivalent_iterations"], 2), "launches", st["gpu_launches"], flush=True)
