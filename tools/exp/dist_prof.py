"""Profile target: one partitioned C4 solve on G emulated ranks (one process, one host thread per
rank, sharing cuda:0) for the ncu launch list of the multi-GPU kernels (compaction into the peer
inboxes, inbox apply, ring kernels) next to k_cycle<DIST>.
    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/exp/dist_prof.py c4 2 [dist_async]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import run_local_group
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
da = len(sys.argv) > 3 and sys.argv[3] == "dist_async"
src, dst, n = digen.make(cfg)


def fn(r, grp):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = di.Graph(src, dst, n, rank=r, world=G, group=grp, stream=s)
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, dist_async=da)
        g.free()
    return st


st = run_local_group(G, fn)[0]
print(cfg, "G", G, "dist_async" if da else "sync", "cycles", st["sweeps"], "eq", round(st["equivalent_iterations"], 2),
      "exchange MB/rank", round(st["exchange_bytes"] / 1e6, 1), "peer-memory sweeps", st["p2p_exchanges"])
