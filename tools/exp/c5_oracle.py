"""North_star parity at full C5 scale on ONE GPU: DI-SOP (asynchronous cycles) on the B200 vs
the sequential CPU oracle (§2.5.5 exactly, one core), both to ||F||_1 <= 1e-10."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import oracle
import paper_1204_6255_b200 as di
D, TOL = 0.85, 1e-10
t = time.time()
src, dst, n = digen.make("c5")
print("C5: N =", n, "L =", len(src), "generated in", round(time.time() - t, 1), "s", flush=True)
g = di.Graph(src, dst, n)
st = g.solve(d=D, tol=TOL, asynchronous=True, graph_loop=True)
st = g.solve(d=D, tol=TOL, asynchronous=True, graph_loop=True)
H = g.history().cpu().numpy()
print("GPU: solve %.1f ms, %d cycles, %.2f eq-iter, residual %.3e, converged %d"
      % (st["solve_ms"], st["sweeps"], st["equivalent_iterations"], st["residual_l1"], st["converged"]), flush=True)
g.free()
torch.cuda.empty_cache()
t = time.time()
Ho, Fo, sto = oracle.di(src, dst, n, d=D, tol=TOL, variant="sop")
secs = time.time() - t
print("oracle (1 core, sequential DI-SOP incl. adjacency build): %.1f s, %d cycles, %.2f nb-iter, residual %.3e"
      % (secs, sto["cycles"], sto["diffusions"] / len(src), float(Fo.sum())), flush=True)
diff = float(np.abs(H - Ho).sum())
print("||H_gpu - H_oracle||_1 = %.3e  (north_star bound 1e-9; G19 guarantee 2*tol/(1-d) = %.3e)"
      % (diff, 2 * TOL / (1 - D)), flush=True)
print("PASS" if diff <= 1e-9 else "FAIL", flush=True)
