"""Experiment: the bench's e2e step, phase by phase, repeated (host link list -> H on host)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make(sys.argv[1] if len(sys.argv) > 1 else "c4")
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
H_host = torch.empty(n, dtype=torch.float64).pin_memory()
stream = torch.cuda.current_stream()
for k in range(5):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = di.Graph(src_p, dst_p, n, stream=stream); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True); t2 = time.perf_counter()
    H = g.history(); H_host.copy_(H, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    g.free(); del H; torch.cuda.synchronize(); t4 = time.perf_counter()
    print("e2e: upload %.1f solve %.1f (dev %.1f) H->host %.1f | free %.1f ms" % ((t1 - t) * 1e3, (t2 - t1) * 1e3, st["solve_ms"], (t3 - t2) * 1e3, (t4 - t3) * 1e3), file=sys.stderr, flush=True)
