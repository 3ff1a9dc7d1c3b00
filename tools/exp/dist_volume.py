"""Experiment: exchange volume of the partitioned solve (emulated ranks on one GPU): entries
(12 B each) per rank per cycle vs the dense alternative, for bulk sweeps and asynchronous cycles.
The volume is a property of the partition and the schedule, not of the interconnect."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import run_local_group
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
Gs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
src, dst, n = digen.make(cfg)
for G in Gs:
    for asyn in (False, True):
        def fn(r, grp):
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                g = di.Graph(src, dst, n, rank=r, world=G, group=grp, stream=s)
                st = g.solve(d=0.85, tol=1e-10, asynchronous=asyn)
                out = (g.lo, g.hi, st)
                g.free()
            return out
        t = time.time()
        res = run_local_group(G, fn)
        st = res[0][2]
        ent = [r[2]["exchange_entries"] for r in res]
        cyc = st["sweeps"]
        dense = [(n - (hi - lo)) * 8 for lo, hi, _ in res]
        print(cfg, "G", G, "async" if asyn else "bulk", "cycles", cyc, "eq", round(st["equivalent_iterations"], 2),
              "resid", st["residual_l1"], "sparse MB/cycle/rank max", round(max(ent) * 12 / cyc / 1e6, 1),
              "dense MB/cycle/rank", round(max(dense) / 1e6, 1), "ratio", round(max(ent) * 12 / cyc / max(dense), 3),
              "wall s", round(time.time() - t, 1), flush=True)
