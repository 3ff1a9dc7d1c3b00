"""ncu driver: C5 on one GPU, two asynchronous solves (profile a k_cycle launch of the second)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c5")
g = di.Graph(src, dst, n)
del src, dst
for k in range(2):
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True)
    print(k, st["solve_ms"], st["sweeps"], flush=True)
