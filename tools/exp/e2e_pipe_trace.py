"""Timeline of the pipelined e2e on C4 (producer uploads vs consumer solves), row_sort = 0."""
import os, sys, time, threading, queue
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
di.set_option("row_sort", 0)
GL = "graph" in sys.argv[1:]
src, dst, n = digen.make("c4")
sp, dp = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
dev = torch.device("cuda", 0)
lo, hi = torch.cuda.Stream.priority_range()
ups = [torch.cuda.Stream(dev, priority=lo) for _ in range(3)]
sols = [torch.cuda.Stream(dev, priority=hi) for _ in range(3)]
H = torch.empty(n, dtype=torch.float64).pin_memory()
q = queue.Queue(maxsize=1)
if "--serial-first" in sys.argv:   # as in bench.py: serial e2e steps before the pipeline
    for k in range(8):
        g = di.Graph(sp, dp, n)
        g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
        H.copy_(g.history())
        g.free()
    torch.cuda.synchronize()
if "--trim" in sys.argv:
    from cuda import cudart
    err, pool = cudart.cudaDeviceGetDefaultMemPool(0)
    print("trim", cudart.cudaMemPoolTrimTo(pool, 0), flush=True)
T0 = time.perf_counter()
def ts(): return (time.perf_counter() - T0) * 1e3
def producer():
    torch.cuda.set_device(dev)
    for k in range(7):
        t = ts()
        g = di.Graph(sp, dp, n, stream=ups[k % 3])
        print(f"upload {k}: {t:8.1f} -> {ts():8.1f}", flush=True)
        q.put((k, g))
th = threading.Thread(target=producer); th.start()
for _ in range(7):
    k, g = q.get()
    t = ts()
    g.set_stream(sols[k % 3])
    with torch.cuda.stream(g.stream):
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=GL)
        t2 = ts()
        Hd = g.history()
        H.copy_(Hd, non_blocking=True)
        g.stream.synchronize()
    print(f"   solve {k}: {t:8.1f} -> {t2:8.1f} (device {st['solve_ms']:.1f}) -> H {ts():8.1f}", flush=True)
    g.free()
th.join()
