"""Fourth pass: what distinguishes the slow fresh-process host-drawn upload (614 ms) from the fast
GPU-drawn one (583 ms): the order of the link list or where the arrays land?
  --via-host : GPU-drawn (sorted) links copied to the host, every GPU buffer released, copied back as
               bench.py does (torch's first two allocations), then uploaded
  --shuffle  : GPU-drawn links permuted on the GPU (unsorted input, the tool's placement)"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = "c5"
n = digen.CONFIGS[cfg].n
dev = torch.device("cuda", 0)
s, d, _ = digen.make_range_gpu(cfg, 0, n)
torch.cuda.synchronize()
if "--via-host" in sys.argv:
    sh, dh = s.cpu(), d.cpu()
    del s, d
    torch.cuda.empty_cache()
    print("free after releasing everything: %.1f GiB" % (torch.cuda.mem_get_info()[0] / 2**30), flush=True)
    s, d = sh.to(dev), dh.to(dev)
if "--shuffle" in sys.argv:
    L = s.numel()
    torch.manual_seed(1)
    # block permutation (a full randperm of 2.16e9 int64 is 17 GB: fine on 180 GB)
    p = torch.randperm(L, device=dev)
    s, d = s[p].contiguous(), d[p].contiguous()
    del p
    torch.cuda.empty_cache()
print("free before the upload: %.1f GiB" % (torch.cuda.mem_get_info()[0] / 2**30), flush=True)
g = di.Graph(s, d, n, stream=torch.cuda.current_stream(dev), build_csc=False)
del s, d
for k in range(3):
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop="--host-loop" not in sys.argv)
    print("solve", k, "ms", round(st["solve_ms"], 1), "cycles", st["sweeps"], "eq-iter %.2f" % st["equivalent_iterations"], flush=True)
g.free()
