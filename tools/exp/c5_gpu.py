"""C5 (R-MAT N = 2^27, L ~ 2.16e9) on ONE B200 with the graph drawn on the GPU (digen.make_range_gpu
over the whole range: the same links as digen.make("c5")): timing of the asynchronous DI-SOP solve.
    python tools/exp/c5_gpu.py [--config c5] [--solves 3] [--profile]"""
import argparse, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--cold", type=int, default=-1, help="option cold_bins (-1 auto, 0 off, 1 on)")
ap.add_argument("--cold-tier", type=int, default=0, help="option cold_tier (first-tier nodes)")
ap.add_argument("--cold-shift", type=int, default=0, help="option cold_shift (slice = 2^shift nodes)")
ap.add_argument("--warm", type=int, default=-1, help="option warm (-1 auto, 0 off)")
ap.add_argument("--warm-shift", type=int, default=0, help="option warm_shift (0 auto)")
a = ap.parse_args()
di.set_option("warm", a.warm)
di.set_option("warm_shift", a.warm_shift)
di.set_option("cold_bins", a.cold)
di.set_option("cold_tier", a.cold_tier)
di.set_option("cold_shift", a.cold_shift)
D = 0.85
t = time.time()
n = digen.CONFIGS[a.config].n
s, d, _ = digen.make_range_gpu(a.config, 0, n)
torch.cuda.synchronize()
print(a.config, "cold_bins", a.cold, "cold_tier", a.cold_tier, "cold_shift", a.cold_shift, "warm", a.warm, "warm_shift", a.warm_shift, "generated on the GPU: N =", n, "L =", s.numel(), "in", round(time.time() - t, 1), "s", flush=True)
t = time.time()
g = di.Graph(s, d, n)
torch.cuda.synchronize()
del s, d
print("build", round(time.time() - t, 2), "s", flush=True)
for k in range(a.solves):
    st = g.solve(d=D, tol=1e-10, asynchronous=True, graph_loop=not a.profile, profile=a.profile)
    print("solve", k, "ms", round(st["solve_ms"], 1), "cycles", st["sweeps"],
          "ms/cycle", round(st["solve_ms"] / max(st["sweeps"], 1), 2),
          "eq-iter", round(st["equivalent_iterations"], 2), "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1),
          "counted GB/s", round(st["counted_bytes"] / st["solve_ms"] / 1e6, 1),
          "residual", st["residual_l1"], "converged", st["converged"], flush=True)
    if a.profile:
        print("   k_cycle avg ms", round(st["push_ms"] / max(st["push_launches"], 1), 3),
              "counted frac", round(st["counted_bytes"] / (st["push_ms"] * 1e-3) / 1e9 / 6550.4, 4), flush=True)
g.free()
