"""Why bench.py --config c5 times the one-GPU C5 solve ~5 % slower than tools/exp/c5_gpu.py
(623.8 vs 592.9 ms on the same box): bench.py's ingredients added one at a time to the plain
solve. Prints the solve time after each.
    python tools/exp/c5_bench_diff.py [--config c5]"""
import argparse, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--skip0", action="store_true", help="no GPU-drawn graph first: the host-drawn upload populates a fresh pool")
a = ap.parse_args()
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)


def solves(g, tag, k=2, **kw):
    for _ in range(k):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True, **kw)
        e1.record(stream)
        e1.synchronize()
        print(f"{tag}: {e0.elapsed_time(e1):.1f} ms (lib {st['solve_ms']:.1f}), {st['sweeps']} cycles, "
              f"{st['equivalent_iterations']:.2f} eq-iter, free {torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB",
              flush=True)


n = digen.CONFIGS[a.config].n
# [0] the tool's path: links drawn on the GPU
if not a.skip0:
    s, d, _ = digen.make_range_gpu(a.config, 0, n)
    g = di.Graph(s, d, n)
    del s, d
    solves(g, "[0] GPU-drawn links, device upload")
    g.free()
    torch.cuda.empty_cache()
# [1] bench.py's path: links drawn on the host, copied, device upload
t = time.time()
src, dst, n = digen.make(a.config, seed=1)
print("host generator", round(time.time() - t, 1), "s", src.dtype, flush=True)
s_d = torch.from_numpy(src).to(dev)
t_d = torch.from_numpy(dst).to(dev)
g = di.Graph(s_d, t_d, n, stream=stream, build_csc=False)
del s_d, t_d
solves(g, "[1] host-drawn links, device upload")
# [2] + the flush buffer
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
flush.fill_(1)
solves(g, "[2] + 512 MiB flush buffer")
# [3] + the clocks sampler
with bench.Clocks(0):
    solves(g, "[3] + nvidia-smi sampler")
# [4] + a profiled host-loop solve in between
g.solve(d=0.85, tol=1e-10, asynchronous=True, profile=True)
solves(g, "[4] after a profiled host-loop solve")
# [5] torch's cache released
torch.cuda.empty_cache()
solves(g, "[5] after torch.cuda.empty_cache()")
g.free()
