"""Per-cycle links (sweep log) and per-CTA cycle spans (option cycle_times) of the C4 bench solve."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c4")
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
st = g.solve(d=0.85, tol=1e-10, asynchronous=True, trace=True)
log = g.sweep_log()
L = g.n_links
print("cycles", st["sweeps"], "ms", round(st["solve_ms"], 2))
for k in range(len(log["r"])):
    print(k, "r %.3e" % log["r"][k], "links/L %.3f" % (log["links"][k] / L), "selected", int(log["selected"][k]))

di.set_option("cycle_times", 1)
g2 = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
st = g2.solve(d=0.85, tol=1e-10, asynchronous=True, profile=True)
print("profiled: push_ms", round(st["push_ms"], 2), "launches", st["push_launches"])
