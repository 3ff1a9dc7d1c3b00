"""(Round-1 experiment: some knobs it sets no longer exist; kept as the record of that run.)
Experiment: k_push occupancy (DI_PUSH_OCC) and red hint on C4 block-ordered solve."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
src, dst, n = digen.make(cfg)
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
CASES = [(4, 1, 4096, 0), (4, 1, 4096, 1), (4, 1, 16384, 0), (4, 1, 16384, 1), (4, 1, 2048, 1), (4, 1, 8192, 1)]
for occ, hint, stripes, rot in CASES:
    os.environ["DI_STRIPE_ROT"] = str(rot)
    __import__("paper_1204_6255_b200").set_option("push_occ", float(str(occ)))
    __import__("paper_1204_6255_b200").set_option("red_hint", float(str(hint)))
    __import__("paper_1204_6255_b200").set_option("stripes", float(str(stripes)))
    g = di.Graph(s_d, t_d, n)
    for K in (1, 8):
        g.solve(d=0.85, tol=1e-10, blocks=K)
        sts = [g.solve(d=0.85, tol=1e-10, blocks=K, profile=p) for p in (False, False, True)]
        st = min(sts[:2], key=lambda s: s["solve_ms"])
        pr = sts[2]
        print(cfg, "rot", rot, "occ", occ, "hint", hint, "stripes", stripes, "K", K, "ms", round(st["solve_ms"], 2),
              "eq", round(st["equivalent_iterations"], 2), "push_ms", round(pr["push_ms"], 1), "select_ms", round(pr["select_ms"], 1), flush=True)
    g.free()
