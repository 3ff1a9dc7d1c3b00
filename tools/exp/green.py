"""Experiment: SM partitions with green contexts (cuda-python driver API) for the library's streams.
(1) the C4 solve on a green-context stream of K SMs; (2) a C4 upload (host link list) on a
partition of the remaining SMs; (3) both at once."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import cuda.bindings.driver as drv
import digen
import paper_1204_6255_b200 as di


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


torch.cuda.init()
torch.zeros(1, device="cuda")
dev = ck(drv.cuDeviceGet(0))
res = ck(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("SMs", res.sm.smCount, flush=True)


def green_stream(n_sm):
    """a green context holding n_sm SMs (split from the device), and a stream in it"""
    r = drv.cuDevSmResourceSplitByCount(1, res, 0, n_sm)
    if int(r[0]) != 0:
        raise RuntimeError(str(r[0]))
    groups = r[1]          # (err, result[], nbGroups, remaining)
    desc = ck(drv.cuDevResourceGenerateDesc([groups[0]], 1))
    g = ck(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = ck(drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    return g, torch.cuda.ExternalStream(int(st))


src, dst, n = digen.make("c4")
s_d, t_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
src_p, dst_p = torch.from_numpy(src).pin_memory(), torch.from_numpy(dst).pin_memory()
full = torch.cuda.Stream()
for k_sm in (148, 112, 96, 80, 64):
    try:
        st = full if k_sm == 148 else green_stream(k_sm)[1]
        g = di.Graph(s_d, t_d, n, stream=st)
        for r in range(3):
            x = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=False)
        print(f"solve on {k_sm} SMs: {x['solve_ms']:.2f} ms, cycles {x['sweeps']}", flush=True)
        g.free()
    except Exception as e:
        print("solve on", k_sm, "failed:", e, flush=True)
for k_sm in (148, 84, 68, 52):
    try:
        st = full if k_sm == 148 else green_stream(k_sm)[1]
        ts = []
        for r in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            g = di.Graph(src_p, dst_p, n, stream=st)
            st.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
            g.free()
        print(f"upload on {k_sm} SMs: {min(ts):.1f} ms", flush=True)
    except Exception as e:
        print("upload on", k_sm, "failed:", e, flush=True)

# both at once: the solve of a resident graph on a partition of A SMs while a host-list upload runs
# on the other 148 - A (the pipelined e2e's two halves)
for A in (112, 96, 80):
    try:
        gs, ss = green_stream(A)
        # the other partition: split the remainder (the split above takes the first A SMs)
        r = drv.cuDevSmResourceSplitByCount(1, res, 0, A)
        rem = r[3]
        desc = ck(drv.cuDevResourceGenerateDesc([rem], 1))
        gu = ck(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        us = torch.cuda.ExternalStream(int(ck(drv.cuGreenCtxStreamCreate(gu, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))))
        g = di.Graph(s_d, t_d, n, stream=ss)
        g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=True)
        import threading
        out = {}
        def up():
            torch.cuda.set_device(0)
            t0 = time.perf_counter()
            gg = di.Graph(src_p, dst_p, n, stream=us)
            us.synchronize()
            out["up"] = (time.perf_counter() - t0) * 1e3
            gg.free()
        th = threading.Thread(target=up)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th.start()
        x = g.solve(d=0.85, tol=1e-10, asynchronous=True, graph_loop=False)
        ts = (time.perf_counter() - t0) * 1e3
        th.join()
        tt = (time.perf_counter() - t0) * 1e3
        print(f"concurrent: solve on {A} SMs {x['solve_ms']:.1f} ms (wall {ts:.1f}), upload on {148 - A} SMs {out['up']:.1f} ms, both {tt:.1f} ms", flush=True)
        g.free()
    except Exception as e:
        print("concurrent", A, "failed:", repr(e), flush=True)
