"""compute-sanitizer driver: every solve path on small graphs (C1 and a loop/duplicate graph)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import run_local_group
graphs = [digen.make("c1", seed=1), digen.small_random(5, n_max=3000)]
for src, dst, n in graphs:
    g = di.Graph(src, dst, n, build_csc=True)
    for kw in (dict(), dict(mode="pull"), dict(mode="auto"), dict(blocks=4), dict(asynchronous=True),
               dict(asynchronous=True, graph_loop=True), dict(graph_loop=True), dict(variant="cyc"),
               dict(variant="pi"), dict(variant="pi_push"), dict(variant="gs")):
        st = g.solve(d=0.85, tol=1e-10, **kw)
        print(n, kw, st["converged"], st["sweeps"], flush=True)
    g.free()
    def fn(r, grp):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            h = di.Graph(src, dst, n, rank=r, world=2, group=grp, stream=s)
            out = [h.solve(d=0.85, tol=1e-10, asynchronous=a)["converged"] for a in (False, True)]
            h.free()
        return out
    print("dist", run_local_group(2, fn), flush=True)
print("done")
