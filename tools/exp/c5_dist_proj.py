"""Per-GPU projection of the partitioned north_star workload (VERDICT r1 "Next round" 4): C5 (N = 2^27,
L = 2.16e9) on G emulated ranks sharing ONE B200, every rank drawing its own source range on the GPU
(digen.make_range_gpu, equal node ranges, DI_LOCAL_LINKS), asynchronous cycles through peer memory
with the compact remote path (hot remote accumulator + cold records). Under ncu the ranks' kernels
serialise, so one rank's k_cycle<DIST> / k_compact_remote / k_apply_inbox durations are what one GPU
of a G-GPU run would spend (the emulated ranks' wall time is not a multi-GPU time).
    python tools/exp/c5_dist_proj.py [G] [config] [--check]   (--check: saves the assembled H)
    python tools/exp/c5_dist_proj.py --one-gpu [config]         (1-GPU solve, compared with it;
                                                                 a fresh process: the first one's
                                                                 memory pool keeps its buffers)"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import assemble, run_local_group
G = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "--one-gpu" else 8
cfg = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "c5"
check = "--check" in sys.argv
if "--parts" in sys.argv:
    di.set_option("dist_parts", int(sys.argv[sys.argv.index("--parts") + 1]))
if "--remote-tier" in sys.argv:
    di.set_option("remote_tier", int(sys.argv[sys.argv.index("--remote-tier") + 1]))
ALPHA = float(sys.argv[sys.argv.index("--alpha") + 1]) if "--alpha" in sys.argv else 1.0   # F4 threshold scale
D, TOL = 0.85, 1e-10
n = digen.CONFIGS[cfg].n
ranges = digen.node_ranges(n, G)
PATH = "/tmp/di_%s_hpart.npy" % cfg
if len(sys.argv) > 1 and sys.argv[1] == "--one-gpu":   # the 1-GPU solve vs the saved partitioned H
    s, t, _ = digen.make_range_gpu(cfg, 0, n)
    g = di.Graph(s, t, n)
    del s, t
    st = g.solve(d=D, tol=TOL, asynchronous=True, graph_loop=True)
    H1 = g.history().cpu().numpy()
    print("1 GPU: %.1f ms, %d cycles, %.2f eq-iter" % (st["solve_ms"], st["sweeps"], st["equivalent_iterations"]), flush=True)
    H = np.load(PATH)
    diff = float(np.abs(H - H1).sum())
    print("||H_partitioned - H_1gpu||_1 = %.3e (bound 2e-10/(1-d) = %.3e) %s" % (diff, 2e-10 / (1 - D),
          "PASS" if diff <= 2e-10 / (1 - D) else "FAIL"), flush=True)
    sys.exit(0)


import threading
GEN = threading.Lock()


def rank(r, grp):
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        lo, hi = ranges[r]
        with GEN:   # one rank at a time; torch's cache returned for libdi's pool afterwards
            s, t, _ = digen.make_range_gpu(cfg, lo, hi)
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        t0 = time.time()
        gr = di.Graph(s, t, n, rank=r, world=G, group=grp, stream=stream, local_range=(lo, hi))
        torch.cuda.synchronize()
        tb = time.time() - t0
        del s, t
        if ALPHA != 1.0:
            gr.set_threshold_scale(ALPHA)
        st = gr.solve(d=D, tol=TOL, asynchronous=True)
        out = ((gr.lo, gr.hi), gr.history().cpu().numpy() if check else None, st, tb, gr.n_links)
        gr.free()
    return out


res = run_local_group(G, rank, timeout=3000)
st = res[0][2]
cyc = max(1, st["sweeps"])
print("remote_tier", di.get_option("remote_tier"), "alpha", ALPHA)
print("%s on %d emulated ranks: build %.1f s, %d cycles, %.2f eq-iter, residual %.3e, converged %d" %
      (cfg, G, max(x[3] for x in res), st["sweeps"], st["equivalent_iterations"], st["residual_l1"], st["converged"]), flush=True)
for r, x in enumerate(res):
    s_ = x[2]
    print("  rank %d: links %d, exchange per cycle: %.1f MB (%d compact 12-B entries, %d cold 16-B records)" %
          (r, x[4], s_["exchange_bytes"] / cyc / 1e6, s_["exchange_entries"] // cyc, s_["exchange_cold"] // cyc), flush=True)
if check:
    np.save(PATH, assemble([x[1] for x in res], [x[0] for x in res], n))
