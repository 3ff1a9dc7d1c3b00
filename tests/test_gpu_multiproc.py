"""The partitioned solve with one process per GPU over NCCL, as bench.py --gpus N
runs it: needs at least two GPUs, skipped otherwise (this round's boxes have one; the emulated
ranks of tests/test_gpu_dist.py cover every kernel and the protocol there). On a multi-GPU box it
checks, against the oracle, the synchronous cycles with the lists written through peer memory
(NCCL symmetric window) and through send/recv, the dense fallback, and the asynchronous
multi-GPU cycles (F2)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = 0.85


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [dict(asynchronous=True), dict(asynchronous=True, p2p=False), dict(exchange="dense"),
         dict(asynchronous=True, dist_async=True), dict()]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as tdist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        tdist.init_process_group("nccl", rank=rank, world_size=world,
                                 device_id=torch.device("cuda", rank))
        import digen
        import paper_1204_6255_b200 as di
        from paper_1204_6255_b200.dist import gather_to_rank0, nccl_rendezvous
        r, w, nid = nccl_rendezvous()
        src, dst, n = digen.make("c1", seed=1)
        g = di.Graph(src, dst, n, rank=r, world=w, nccl_id=nid)
        out = []
        for kw in CASES:
            st = g.solve(d=D, tol=1e-10, variant="sop", **kw)
            H = gather_to_rank0(g.history().cpu().numpy(), g.lo, g.hi, n)
            out.append((kw, st, None if H is None else H.tolist()))
        g.free()
        # DI_LOCAL_LINKS: this process passes only its own sources' links (equal node ranges)
        lo, hi = n * r // w, n * (r + 1) // w
        m = (src >= lo) & (src < hi)
        gl = di.Graph(src[m], dst[m], n, rank=r, world=w, nccl_id=nid, local_range=(lo, hi))
        st = gl.solve(d=D, tol=1e-10, variant="sop", asynchronous=True)
        H = gather_to_rank0(gl.history().cpu().numpy(), gl.lo, gl.hi, n)
        out.append((dict(local_links=True), st, None if H is None else H.tolist()))
        gl.free()
        q.put((rank, out))
        tdist.barrier()
        tdist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error: " + repr(e)))


def test_nccl_multiprocess_partitioned():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU over NCCL)")
    import digen
    import oracle
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(60)
    for r, o in res.items():
        assert not isinstance(o, str), o
    src, dst, n = digen.make("c1", seed=1)
    Ho, _, _ = oracle.di(src, dst, n, d=D, tol=1e-10, variant="sop")
    for k, kw in enumerate(CASES + [dict(local_links=True)]):
        sts = [res[r][k][1] for r in range(world)]
        assert all(s["converged"] == 1 for s in sts), (kw, sts)
        assert len({s["link_diffusions"] for s in sts}) == 1, kw   # global counters
        H = np.array(res[0][k][2])
        assert np.abs(H - Ho).sum() <= 1e-9, kw
        if kw.get("p2p", True) and kw.get("exchange") != "dense":
            assert sts[0]["p2p_exchanges"] > 0 or sts[0]["exchange_entries"] > 0, kw
