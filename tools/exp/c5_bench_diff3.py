"""Third pass: does the memory torch holds when libdi's pool is first populated matter? GPU-drawn C5
links; --empty releases torch's cache (the generator's ~90 GB of temporaries) before the upload, as in
bench.py where torch holds only the 17.3 GB link list."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = "c5"
n = digen.CONFIGS[cfg].n
s, d, _ = digen.make_range_gpu(cfg, 0, n)
torch.cuda.synchronize()
if "--empty" in sys.argv:
    torch.cuda.empty_cache()
print("free before the upload: %.1f GiB" % (torch.cuda.mem_get_info()[0] / 2**30), flush=True)
g = di.Graph(s, d, n)
del s, d
for k in range(3):
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    print("solve", k, "ms", round(st["solve_ms"], 1), "cycles", st["sweeps"], "free %.1f GiB" % (torch.cuda.mem_get_info()[0] / 2**30), flush=True)
g.free()
