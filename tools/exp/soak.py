"""Soak: repeated asynchronous solves (host loop and device-side graph loop) on C2/C3/C4, every
one checked for convergence, residual and the conservation identity; catches rare hazards of the
hub-item flag and the persistent-kernel protocol."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c2,c3,c4").split(","):
    src, dst, n = digen.make(cfg)
    outd = np.bincount(src, minlength=n)
    g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n)
    t = time.time()
    ms = []
    for k in range(reps):
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=(k % 2 == 1))
        assert st["converged"] == 1 and st["residual_l1"] <= 1e-10, (cfg, k, st)
        ms.append(st["solve_ms"])
        if k % 10 == 0:
            H = g.history().cpu().numpy()
            l1f, F = g.residual(return_F=True)
            F = F.cpu().numpy()
            cons = F.sum() + 0.15 * H[outd > 0].sum() + H[outd == 0].sum()
            assert abs(cons - 0.15) <= 1e-12 and np.all(F >= 0), (cfg, k, cons)
    print(cfg, reps, "solves ok, ms min/median/max", round(min(ms), 2), round(float(np.median(ms)), 2),
          round(max(ms), 2), "wall", round(time.time() - t, 1), "s", flush=True)
    g.free()
