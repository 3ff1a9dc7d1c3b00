"""(Round-1 experiment: some knobs it sets no longer exist; kept as the record of that run.)
Experiment: k_push (0) vs k_push_b (1): solve time on a config for K in a list; H agreement."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
Ks = [int(k) for k in (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")]
src, dst, n = digen.make(cfg)
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
Hs = {}
for kern in (0, 1):
    os.environ["DI_PUSH_KERNEL"] = str(kern)
    g = di.Graph(s_d, t_d, n)
    for K in Ks:
        g.solve(d=0.85, tol=1e-10, blocks=K)
        sts = [g.solve(d=0.85, tol=1e-10, blocks=K, profile=p) for p in (False, False, True)]
        st = min(sts[:2], key=lambda s: s["solve_ms"])
        pr = sts[2]
        Hs[(kern, K)] = g.history()
        print(cfg, "kernel", kern, "K", K, "ms", round(st["solve_ms"], 2), "sweeps", st["sweeps"],
              "eq", round(st["equivalent_iterations"], 2), "push_ms", round(pr["push_ms"], 1),
              "select_ms", round(pr["select_ms"], 1), "push GB/s", round(pr["push_bytes"] / pr["push_ms"] / 1e6, 1),
              "resid", st["residual_l1"], flush=True)
    g.free()
for K in Ks:
    print("L1(H0-H1) K", K, float((Hs[(0, K)] - Hs[(1, K)]).abs().sum()))
