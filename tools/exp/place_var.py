"""Experiment: solve-time variance across repeated uploads (allocation placement)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c4")
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
keep = []
for k in range(8):
    if k % 2 == 1:
        keep.append(torch.empty((k + 1) * (64 << 20), dtype=torch.uint8, device="cuda"))  # shift torch's arena
    g = di.Graph(s_d if k < 4 else src_p, t_d if k < 4 else dst_p, n)
    ts = [g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)["solve_ms"] for _ in range(3)]
    print(k, "device" if k < 4 else "host", "solve ms", [round(t, 2) for t in ts], flush=True)
    g.free()
