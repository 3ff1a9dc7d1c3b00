"""Experiment: where the e2e upload outliers come from. (1) raw H2D copies of the C4 link list from
pinned host memory (torch copy_), (2) host-pointer uploads with the build_trace phases."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c4")
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
s_d, t_d = torch.empty_like(src_p, device="cuda"), torch.empty_like(dst_p, device="cuda")
for k in range(8):
    torch.cuda.synchronize(); t = time.perf_counter()
    s_d.copy_(src_p, non_blocking=True); t_d.copy_(dst_p, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("raw H2D %.1f ms (%.1f GB/s)" % (dt * 1e3, 8 * src.size / dt / 1e9), flush=True)
del s_d, t_d
torch.cuda.empty_cache()
di.set_option("build_trace", 1)
for k in range(10):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = di.Graph(src_p, dst_p, n); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    g.free(); torch.cuda.synchronize()
    print("upload %.1f ms" % ((t1 - t) * 1e3), file=sys.stderr, flush=True)
