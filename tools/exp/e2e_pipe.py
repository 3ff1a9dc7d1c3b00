"""e2e on C4 through the public API, serial and pipelined (bench.py's e2e_pipelined), per builder:
    python tools/exp/e2e_pipe.py"""
import os, sys, time, types
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c4")
sp, dp = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
dev = torch.device("cuda", 0)
args = types.SimpleNamespace(e2e_steps=5, variant="sop")
H = torch.empty(n, dtype=torch.float64).pin_memory()
for rs in (0, 1):
    di.set_option("row_sort", rs)
    ms, lk = [], 0
    for k in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = di.Graph(sp, dp, n)
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
        H.copy_(g.history())
        torch.cuda.synchronize()
        if k >= 1:
            ms.append((time.perf_counter() - t) * 1e3)
            lk += st["link_diffusions"]
        g.free()
    print(f"row_sort={rs} serial: {sum(ms) / len(ms):.1f} ms/step, {lk / (sum(ms) * 1e-3) / 1e9:.1f} GTEPS", flush=True)
    p = bench.e2e_pipelined(di, sp, dp, n, dev, args, True, True)
    print(f"row_sort={rs} pipelined: {p}", flush=True)
