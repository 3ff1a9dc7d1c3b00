"""N > 1 host path on CPU (world_size 2, gloo): the NCCL-id rendezvous, slice assembly and the
loud failure of a partitioned upload without a GPU. The partitioned sweeps themselves are
covered on the GPU by tests/test_gpu_dist.py (emulated ranks)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as tdist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1204_6255_b200 as di
        from paper_1204_6255_b200.dist import gather_to_rank0, nccl_rendezvous
        r, w, nid = nccl_rendezvous()
        ids = [None] * w
        tdist.all_gather_object(ids, nid)
        # slices of a 10-node vector with uneven ranges, assembled on rank 0
        bounds = [0, 3, 10]
        lo, hi = bounds[r], bounds[r + 1]
        full = gather_to_rank0(np.arange(lo, hi, dtype=np.float64) * 0.5, lo, hi, 10)
        # a partitioned upload without a CUDA device must fail loudly (no CPU fallback)
        err = None
        if not torch.cuda.is_available():
            try:
                di.Graph(np.array([0, 1], np.int32), np.array([1, 0], np.int32), 2,
                         rank=r, world=w, nccl_id=nid)
            except RuntimeError as e:   # DIError (DI_ECUDA / DI_ENCCL) or torch's "no driver"
                err = getattr(e, "status", "raised")
        q.put((rank, r, w, ids, None if full is None else full.tolist(), err, torch.cuda.is_available()))
        tdist.barrier()
        tdist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e)))


def test_gloo_world2_rendezvous_and_assembly():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(60)
    for o in out:
        assert o[1] != "error", o
    out.sort()
    for rank, r, w, ids, full, err, cuda in out:
        assert r == rank and w == 2
        assert len(ids) == 2 and ids[0] == ids[1] and len(ids[0]) == 128
        if not cuda:
            assert err in (-3, -4, "raised")   # loud failure, never a silent CPU path
    assert out[0][4] == (np.arange(10) * 0.5).tolist()
    assert out[1][4] is None


def test_assemble_checks_ranges():
    from paper_1204_6255_b200.dist import assemble
    v = assemble([np.array([1.0, 2.0]), np.array([3.0])], [(0, 2), (2, 3)], 3)
    assert v.tolist() == [1.0, 2.0, 3.0]
    with pytest.raises(ValueError):
        assemble([np.array([1.0]), np.array([3.0])], [(0, 1), (2, 3)], 3)
    with pytest.raises(ValueError):
        assemble([np.array([1.0, 2.0])], [(0, 2)], 3)
