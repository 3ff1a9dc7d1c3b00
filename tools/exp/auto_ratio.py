"""Experiment: DI_AUTO push/pull threshold on C4 (solve time, pull sweeps, per-sweep density)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import digen
src, dst, n = digen.make(sys.argv[1] if len(sys.argv) > 1 else "c4")
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
import paper_1204_6255_b200 as di
res = {}
for ratio in [0.35, 0.5, 0.65, 0.8, 2.0]:
    __import__("paper_1204_6255_b200").set_option("auto_ratio", float(str(ratio)))
    g = di.Graph(s_d, t_d, n, build_csc=True)
    g.solve(d=0.85, tol=1e-10, mode="auto")
    ts = []
    for _ in range(3):
        st = g.solve(d=0.85, tol=1e-10, mode="auto", trace=True, profile=True)
        ts.append(st["solve_ms"])
    log = g.sweep_log()
    res[ratio] = dict(ms=min(ts), sweeps=st["sweeps"], pull=st["pull_sweeps"], push_ms=st["push_ms"], select_ms=st["select_ms"])
    print(ratio, res[ratio], flush=True)
    if ratio == 0.35:
        print("density", np.round(log["links"] / len(src), 3).tolist(), flush=True)
    g.free()
