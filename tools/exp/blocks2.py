"""(Round-1 experiment: some knobs it sets no longer exist; kept as the record of that run.)
Experiment: block-ordered cycles with push / pull / auto sub-sweeps (+ agreement of H)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import time
import torch
import digen
import paper_1204_6255_b200 as di
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
Ks = [int(k) for k in (sys.argv[2] if len(sys.argv) > 2 else "8").split(",")]
ratios = [float(r) for r in (sys.argv[3] if len(sys.argv) > 3 else "0.5").split(",")]
src, dst, n = digen.make(cfg)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=True)
ref = None
for K in Ks:
    for mode in ("push", "pull", "auto"):
        for ratio in (ratios if mode == "auto" else [None]):
            if ratio is not None:
                os.environ["DI_AUTO_RATIO_BLK"] = str(ratio)
                g.free(); g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=True)
            t = time.time()
            g.solve(d=0.85, tol=1e-10, blocks=K, mode=mode)
            tb = time.time() - t
            sts = [g.solve(d=0.85, tol=1e-10, blocks=K, mode=mode, profile=p) for p in (False, False, True)]
            st = min(sts[:2], key=lambda s: s["solve_ms"])
            pr = sts[2]
            H = g.history()
            if ref is None:
                ref = H.clone()
            print(cfg, "K", K, mode, ratio, "ms", round(st["solve_ms"], 2), "cycles", st["sweeps"],
                  "eq", round(st["equivalent_iterations"], 2), "pulled", st["pull_sweeps"],
                  "diffuse_ms", round(pr["push_ms"], 1), "select_ms", round(pr["select_ms"], 1),
                  "resid", st["residual_l1"], "dH", float((H - ref).abs().sum()), "first", round(tb, 1), flush=True)
