"""Multi-GPU plumbing for the partitioned solve: rendezvous and slice assembly.

Marshalling only — the partition, the sweeps and the fluid exchange run inside libdi.so.

* One process per GPU: ``rank, world, nccl_id = nccl_rendezvous()`` under torch.distributed
  (rank 0 draws the ncclUniqueId through libdi, every rank receives the same 128 bytes), then
  ``Graph(src, dst, n, rank=rank, world=world, nccl_id=nccl_id)`` on every rank.
* Emulated ranks on one GPU: ``run_local_group(world, fn)`` runs fn(rank, group) on one host
  thread per rank with a shared LocalGroup; a failing rank aborts the group so the others return
  instead of waiting at a collective.
* ``assemble(slices)``: the node ranges are contiguous in the caller's numbering and ordered by
  rank, so the global vector is the rank-ordered concatenation of the per-rank slices.
"""
from __future__ import annotations

import threading

import numpy as np


def nccl_rendezvous(group=None):
    """(rank, world, nccl_id bytes) for the current torch.distributed process group."""
    import torch.distributed as tdist

    from . import nccl_unique_id
    rank, world = tdist.get_rank(group), tdist.get_world_size(group)
    box = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(box, src=0, group=group)
    nid = box[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("nccl_rendezvous: bad unique id broadcast")
    return rank, world, bytes(nid)


def assemble(slices, ranges=None, n=None):
    """Concatenate per-rank slices (rank order). With ranges [(lo, hi), ...], check that they tile
    [0, n) contiguously and that every slice has its range's length."""
    slices = [np.asarray(s) for s in slices]
    if ranges is not None:
        pos = 0
        for (lo, hi), s in zip(ranges, slices):
            if lo != pos or hi < lo or len(s) != hi - lo:
                raise ValueError(f"slice ranges do not tile [0, n): {ranges}")
            pos = hi
        if n is not None and pos != n:
            raise ValueError(f"slice ranges end at {pos}, not {n}")
    return np.concatenate(slices) if slices else np.zeros(0)


def gather_to_rank0(local, lo, hi, n, group=None):
    """torch.distributed gather of this rank's slice (numpy) into the global vector on rank 0
    (None elsewhere). Works with gloo (CPU) and nccl process groups (objects travel as pickles)."""
    import torch.distributed as tdist
    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    out = [None] * world if rank == 0 else None
    tdist.gather_object((int(lo), int(hi), np.asarray(local)), out, dst=0, group=group)
    if rank != 0:
        return None
    return assemble([o[2] for o in out], [(o[0], o[1]) for o in out], n)


def run_local_group(world, fn, timeout=600.0):
    """Run fn(rank, group) for rank in [0, world) on `world` threads sharing one LocalGroup.
    Returns the list of results; re-raises the first failure (after aborting the group)."""
    from . import LocalGroup
    grp = LocalGroup(world)
    results = [None] * world
    errors = []

    def work(r):
        try:
            results[r] = fn(r, grp)
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors.append((r, e))
            grp.abort()

    threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    if any(t.is_alive() for t in threads):
        grp.abort()
        for t in threads:
            t.join(30.0)
        raise TimeoutError(f"run_local_group: ranks still running after {timeout} s")
    if errors:
        raise errors[0][1]
    grp.free()
    return results
