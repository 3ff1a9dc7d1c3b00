"""compute-sanitizer driver for the round-2 kernels (run under `compute-sanitizer --tool memcheck`
and `--tool racecheck`; `tools/exp/sanitize.py` covers the round-1 paths): on small graphs, with the
tiers forced by options, the warm tier of k_cycle (shared-memory accumulators and their flush), the
cold bins (k_cycle<COLD> + k_cold_apply), the LOOPS instantiations, hub items, the compact remote
path of partitioned asynchronous cycles (per-range hot tier, encoded columns, cold records into the
owner's inbox) at 2 and 4 emulated ranks, cycles in parts, the F2 rings, and di_test_cycle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import digen
import paper_1204_6255_b200 as di
from paper_1204_6255_b200.dist import run_local_group


def skewed(seed, n=4096 * 4):
    # hot targets that are hub rows, self-loops on two of them (as tests/test_gpu_solve.py)
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 6 * n).astype(np.int32)
    dst = rng.integers(0, n, 6 * n).astype(np.int32)
    m = len(src)
    for hub, share, out in ((77, 0.04, 9000), (5000, 0.02, 3000), (123, 0.01, 100)):
        k = int(share * m)
        tgt = rng.choice(n, out, replace=False).astype(np.int32)
        src = np.concatenate([src, rng.integers(0, n, k).astype(np.int32), np.full(out, hub, np.int32)])
        dst = np.concatenate([dst, np.full(k, hub, np.int32), tgt])
    src = np.concatenate([src, np.array([77, 5000], np.int32)])
    dst = np.concatenate([dst, np.array([77, 5000], np.int32)])
    return src, dst, n


def check(g, st, tag):
    g.residual()
    g.history()
    print(tag, st["converged"], st["sweeps"], flush=True)
    assert st["converged"] == 1, tag


graphs = [("c1", digen.make("c1", seed=1)), ("loops", digen.small_random(5, n_max=3000)),
          ("skewed", skewed(3))]
for name, (src, dst, n) in graphs:
    # one GPU: warm tier sizes, cold bins with and without the warm tier, both loop drivers
    for opts in (dict(warm=128), dict(warm=4032), dict(warm=0), dict(cold_bins=1, cold_tier=max(1, n // 8)),
                 dict(cold_bins=1, cold_tier=max(1, n // 8), cold_shift=8), dict(long_lanes=0)):
        ctx = [di.option(k, v) for k, v in opts.items()]
        for c in ctx:
            c.__enter__()
        try:
            g = di.Graph(src, dst, n)
        finally:
            for c in reversed(ctx):
                c.__exit__(None, None, None)
        for kw in (dict(asynchronous=True), dict(asynchronous=True, graph_loop=True),
                   dict(asynchronous=True, variant="cyc")):
            check(g, g.solve(d=0.85, tol=1e-10, **kw), (name, opts, kw))
        g.free()
    # the bench kernel's select-and-take in record mode
    g = di.Graph(src, dst, n)
    g.test_cycle(np.full(n, 0.15 / n), np.zeros(n), 0.15)
    g.free()
    # partitioned: compact remote path (default), cycles in parts, rings, the global accumulator
    for world in (2, 4):
        for opts, kw in ((dict(), dict(asynchronous=True)),
                         (dict(remote_tier=max(1, n // (16 * world))), dict(asynchronous=True)),
                         (dict(dist_parts=2), dict(asynchronous=True)),
                         (dict(remote_compact=0), dict(asynchronous=True)),
                         (dict(), dict(asynchronous=True, dist_async=True)),
                         (dict(), dict())):
            def fn(r, grp):
                torch.cuda.set_device(0)
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    h = di.Graph(src, dst, n, rank=r, world=world, group=grp, stream=s)
                    st = h.solve(d=0.85, tol=1e-10, **kw)
                    h.free()
                return st["converged"], st["sweeps"]
            ctx = [di.option(k, v) for k, v in opts.items()]
            for c in ctx:
                c.__enter__()
            try:
                out = run_local_group(world, fn)
            finally:
                for c in reversed(ctx):
                    c.__exit__(None, None, None)
            print(name, "dist", world, opts, kw, out, flush=True)
            assert all(o[0] == 1 for o in out)
print("done")
