"""ncu driver: C5 on one GPU (drawn on the GPU), one asynchronous DI-SOP solve (host loop)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
n = digen.CONFIGS["c5"].n
s, d, _ = digen.make_range_gpu("c5", 0, n)
g = di.Graph(s, d, n)
del s, d
st = g.solve(d=0.85, tol=1e-10, asynchronous=True)
print(st["sweeps"], st["solve_ms"], flush=True)
