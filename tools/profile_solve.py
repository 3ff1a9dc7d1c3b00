"""Minimal driver for ncu: build the config graph, run `--solves` DI solves (first is warm-up).
    ncu ... python tools/profile_solve.py --config c4 --solves 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import digen  # noqa: E402
import paper_1204_6255_b200 as di  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--variant", default="sop")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--mode", default="push")
ap.add_argument("--no-reorder", action="store_true")
ap.add_argument("--blocks", type=int, default=1)
ap.add_argument("--asynchronous", action="store_true")
args = ap.parse_args()
src, dst, n = digen.make(args.config)
g = di.Graph(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), n, build_csc=args.mode != "push",
             reorder=not args.no_reorder)
for k in range(args.solves):
    st = g.solve(d=0.85, tol=1e-10, variant=args.variant, mode=args.mode, blocks=args.blocks,
                 asynchronous=args.asynchronous)
    print(k, st["sweeps"], st["solve_ms"], st["equivalent_iterations"], flush=True)
torch.cuda.synchronize()
