"""Solve time against where the library's arrays land: a pad of X GiB is allocated (and kept) before
anything else, then the config's links are drawn on the GPU (their temporaries released) and uploaded.
    python tools/exp/placement_sweep.py c4 0 2 8 32 64 100"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
if len(sys.argv) > 2 and sys.argv[2] == "--one":
    import torch
    import digen
    import paper_1204_6255_b200 as di
    cfg, pad_gib = sys.argv[1], float(sys.argv[3])
    dev = torch.device("cuda", 0)
    pad = torch.empty(int(pad_gib * 2**30), dtype=torch.uint8, device=dev) if pad_gib > 0 else None
    n = digen.CONFIGS[cfg].n
    s, d, _ = digen.make_range_gpu(cfg, 0, n)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    g = di.Graph(s, d, n)
    del s, d
    ms = []
    for k in range(6):
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
        ms.append(st["solve_ms"])
    print("%s pad %5.1f GiB: solves %s ms, %d cycles, %.2f eq-iter" % (cfg, pad_gib, " ".join("%.2f" % m for m in ms[2:]), st["sweeps"], st["equivalent_iterations"]), flush=True)
    g.free()
else:
    cfg = sys.argv[1]
    for p in sys.argv[2:]:
        subprocess.call([sys.executable, os.path.abspath(__file__), cfg, "--one", p])
