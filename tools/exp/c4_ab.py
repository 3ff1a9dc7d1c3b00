"""A/B of upload-time options on the bench's workload (C4, asynchronous DI-SOP in the graph loop,
512 MiB L2 flush before every solve): python tools/exp/c4_ab.py NAME V1 V2 ... [--config c4]
or combinations: python tools/exp/c4_ab.py warm=4096,warm_flush=8 warm=0 ..."""
import contextlib
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import digen
import paper_1204_6255_b200 as di
args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c4"
if "--config" in sys.argv:
    args.remove(cfg)
if "=" in args[0]:
    combos = [[(kv.split("=")[0], float(kv.split("=")[1])) for kv in a.split(",")] for a in args]
else:
    combos = [[(args[0], float(v))] for v in args[1:]]
src, dst, n = digen.make(cfg)
s, t = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for rep in range(2):
    for combo in combos:
        with contextlib.ExitStack() as es:
            for k_, v_ in combo:
                es.enter_context(di.option(k_, v_))
            g = di.Graph(s, t, n)
        ms = []
        for k in range(6):
            flush.fill_(1)
            st = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
            if k >= 1:
                ms.append(st["solve_ms"])
        st = g.solve(d=0.85, tol=1e-10, asynchronous=True, profile=True)
        kc = st["push_ms"] / max(1, st["push_launches"])
        frac = st["counted_bytes"] / (st["push_ms"] * 1e-3) / 1e9 / 6550.4
        tag = ",".join(f"{k_}={v_:g}" for k_, v_ in combo)
        print(f"{cfg} {tag}: median {statistics.median(ms):.2f} ms (min {min(ms):.2f}), cycles {st['sweeps']}, "
              f"eq-iter {st['equivalent_iterations']:.2f}, GTEPS {st['link_diffusions'] / statistics.median(ms) / 1e6:.1f}, "
              f"k_cycle {kc:.3f} ms, counted frac {frac:.4f}", flush=True)
        g.free()
