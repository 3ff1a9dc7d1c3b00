"""Experiment: upload (build) time, device vs host pointers, repeated; e2e pieces."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make(sys.argv[1] if len(sys.argv) > 1 else "c4")
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
for k in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = di.Graph(s_d, t_d, n); torch.cuda.synchronize(); t1 = time.perf_counter()
    g.free(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("device ptrs: upload %.1f ms, free %.1f ms" % ((t1 - t) * 1e3, (t2 - t1) * 1e3), flush=True)
for k in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = di.Graph(src_p, dst_p, n); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True); t2 = time.perf_counter()
    H = g.history().cpu(); t3 = time.perf_counter()
    g.free(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print("host ptrs: upload %.1f solve %.1f (dev %.1f) history %.1f free %.1f ms" % ((t1 - t) * 1e3, (t2 - t1) * 1e3, st["solve_ms"], (t3 - t2) * 1e3, (t4 - t3) * 1e3), flush=True)
