"""Experiment: node order (relabelling stripes) vs DI_ASYNC work (eq-iter) and time, C4."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
for stripes, reorder in [(int(x), True) for x in (sys.argv[2] if len(sys.argv) > 2 else "4096,1,64,256,16384").split(",")]:
    __import__("paper_1204_6255_b200").set_option("stripes", float(str(stripes)))
    g = di.Graph(s_d, t_d, n, reorder=reorder)
    g.solve(d=0.85, tol=1e-10, asynchronous=True)
    sts = [g.solve(d=0.85, tol=1e-10, asynchronous=True) for _ in range(3)]
    st = min(sts, key=lambda s: s["solve_ms"])
    print(cfg, "stripes", stripes, "reorder", reorder, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"],
          "eq", [round(s["equivalent_iterations"], 2) for s in sts], "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1), flush=True)
    g.free()
