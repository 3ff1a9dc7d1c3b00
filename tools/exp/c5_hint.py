"""Experiment: C5 single GPU, F RED cache hint (DI_RED_HINT) effect on the asynchronous cycle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
src, dst, n = digen.make("c5")
for hint in ("1", "0"):
    __import__("paper_1204_6255_b200").set_option("red_hint", float(hint))
    g = di.Graph(src, dst, n)
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
    print("hint", hint, "ms", round(st["solve_ms"], 1), "cycles", st["sweeps"], "GTEPS", round(st["link_diffusions"] / st["solve_ms"] / 1e6, 1), flush=True)
    g.free()
