"""Experiment: run-to-run variance of the host-pointer upload (the e2e outliers): 12 uploads of C4
from pinned host memory with the build_trace option's phase times."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c4")
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
for k in range(12):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = di.Graph(src_p, dst_p, n); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    g.free(); torch.cuda.synchronize()
    print("upload %.1f ms" % ((t1 - t) * 1e3), file=sys.stderr, flush=True)
