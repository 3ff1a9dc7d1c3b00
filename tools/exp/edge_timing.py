import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from gpu_util import upload
D = 0.85
for n in (1, 1023, 1024, 1025, 4097, 20000):
    rng = np.random.default_rng(n)
    m = 4 * n
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    if n == 20000:
        src = np.concatenate([src, np.zeros(15000, np.int32), np.arange(1, 12001, dtype=np.int32)])
        dst = np.concatenate([dst, np.arange(1, 15001, dtype=np.int32), np.full(12000, 7, np.int32)])
    t = time.time()
    g = upload(src, dst, n, build_csc=True)
    print(n, "upload", round(time.time() - t, 2), flush=True)
    for variant, mode in (("sop", "push"), ("cyc", "push"), ("sop", "pull"), ("sop", "auto")):
        t = time.time()
        st = g.solve(d=D, tol=1e-13, variant=variant, mode=mode)
        print(n, variant, mode, round(time.time() - t, 3), st["sweeps"], st["gpu_launches"], st["solve_ms"], flush=True)
    g.free()
