"""Second pass of tools/exp/c5_bench_diff.py: bench.py's timed loop itself (L2 flush before every
solve, graph-loop and profiled host-loop solves alternating) on GPU-drawn C5 links."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
n = digen.CONFIGS[cfg].n
s, d, _ = digen.make_range_gpu(cfg, 0, n)
g = di.Graph(s, d, n, stream=stream, build_csc=False)
del s, d
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def one(tag, fill, profile, graph, **kw):
    if fill:
        flush.fill_(1)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    st = g.solve(d=0.85, tol=1e-10, variant="sop", profile=profile, mode="push", blocks=1,
                 graph_loop=graph, asynchronous=True, dist_async=False, **kw)
    e1.record(stream)
    e1.synchronize()
    print(f"{tag}: {e0.elapsed_time(e1):.1f} ms (lib {st['solve_ms']:.1f}), {st['sweeps']} cycles", flush=True)


for _ in range(2):
    one("[A] plain graph-loop solve", False, False, True)
for _ in range(3):
    one("[B] flush before the solve", True, False, True)
for _ in range(2):
    one("[C] no flush again", False, False, True)
for _ in range(2):
    one("[D] flush, graph loop", True, False, True)
    one("[D] flush, profiled host loop", True, True, False)
for _ in range(2):
    one("[E] no flush, graph loop", False, False, True)
g.free()
