"""The north_star workload partitioned: C5 (N = 2^27, L = 2.16e9) on G emulated ranks sharing ONE
B200 (one host thread per rank; the fused peer-memory exchange between ranks' inboxes on the same
device), against the single-GPU solve of the same graph (itself checked against the sequential
CPU oracle: profiles/r1_v17_c5_oracle.txt). Times are NOT multi-GPU times (the ranks share the
GPU); the point is the partitioned protocol at full scale: convergence and the H agreement."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import assemble, run_local_group
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
DA = len(sys.argv) > 2 and sys.argv[2] == "dist_async"   # F2: asynchronous multi-GPU cycles
D, TOL = 0.85, 1e-10
t = time.time()
src, dst, n = digen.make("c5")
print("C5: N =", n, "L =", len(src), "generated in", round(time.time() - t, 1), "s", flush=True)
s_d = torch.from_numpy(src).cuda()
d_d = torch.from_numpy(dst).cuda()
del src, dst
g = di.Graph(s_d, d_d, n)
st = g.solve(d=D, tol=TOL, asynchronous=True, graph_loop=True)
H1 = g.history().cpu().numpy()
print("1 GPU: %.1f ms, %d cycles, %.2f eq-iter, residual %.3e" % (st["solve_ms"], st["sweeps"],
      st["equivalent_iterations"], st["residual_l1"]), flush=True)
g.free()
torch.cuda.empty_cache()


def rank(r, grp):
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        t0 = time.time()
        gr = di.Graph(s_d, d_d, n, rank=r, world=G, group=grp, stream=stream)
        tb = time.time() - t0
        st = gr.solve(d=D, tol=TOL, asynchronous=True, dist_async=DA)
        out = ((gr.lo, gr.hi), gr.history().cpu().numpy(), st, tb)
        gr.free()
    return out


t = time.time()
res = run_local_group(G, rank, timeout=1200)
H = assemble([h for _, h, _, _ in res], [rg for rg, _, _, _ in res], n)
st = res[0][2]
diff = float(np.abs(H - H1).sum())
print(("F2 " if DA else "") + "%d emulated ranks: build %.1f s, solve %.1f ms (shared GPU), %d cycles, %.2f eq-iter, residual %.3e, "
      "peer-memory sweeps %d, lists %.1f MB per rank per cycle" % (G, max(x[3] for x in res), st["solve_ms"],
      st["sweeps"], st["equivalent_iterations"], st["residual_l1"], st["p2p_exchanges"],
      max(x[2]["exchange_bytes"] for x in res) / max(1, st["sweeps"]) / 1e6), flush=True)
print("||H_partitioned - H_1gpu||_1 = %.3e (both to 1e-10: bound 2e-10/(1-d) = %.3e)" % (diff, 2e-10 / (1 - D)))
print("PASS" if st["converged"] == 1 and diff <= 2e-10 / (1 - D) else "FAIL", flush=True)
