#!/usr/bin/env python
"""bench.py — D-iteration (arXiv:1204.6255) hot path on B200: GTEPS and time-to-||F||_1 <= 1e-10.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--variant sop] [--impl ours|reference]

A step is one whole solve of the hot path: F = B, H = 0, asynchronous DI-SOP
cycles (one persistent kernel per cycle: select + take + push, R7) until ||F||_1 <= 1e-10,
on the graph resident in HBM (the device CSR build a0 is "Init", timed separately as in PAPER.md
P:61-63, and inside `e2e`). value = link diffusions / solve time (GTEPS = 1e9 link-diffusions/s,
all ranks). The default workload is BASELINE.json configs[3] (C4: R-MAT N=2^24, L~268M, the
largest single-GPU configuration) at every N (strong scaling); --config c5 is the north_star's.
Inputs (col 1.07 GB, F/H 134 MB each) exceed the 126 MB L2, and L2 is additionally flushed
(512 MiB write) before every timed step.

--gpus N > 1 without WORLD_SIZE re-launches this script under torch.distributed.run (one process
per GPU, 127.0.0.1); every rank generates only its own source range on its GPU and uploads it
with DI_LOCAL_LINKS. A process group whose size differs from --gpus is refused.

--impl reference times the CPU oracle (oracle/, sequential DI-SOP exactly as PAPER.md §2.5.5)
on a bounded sample of the same workload (the first cycles of the solve), on this host.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "link-diffusions/sec (GTEPS) and time-to-||F||_1<=1e-10; % HBM roofline"
UNIT = "GTEPS"
RED_PEAK = 192.0   # random fp64 red.global.add into an L2-resident array, tools/micro/atomics.cu
D = 0.85
TOL = 1e-10


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel="k_push"):
    """Per-launch dram bytes of the push kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(kernel)
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = f"/tmp/di_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [l.strip().split(", ") for l in open(self.path) if l.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def make_graph(cfg, seed):
    import digen
    t = time.time()
    src, dst, n = digen.make(cfg, seed=seed)
    return src, dst, n, time.time() - t


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_cmd(gpus, argv, port=None):
    """The torch.distributed.run command that runs this bench with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port or free_port()}",
            os.path.abspath(__file__), *argv]


def spawn(gpus, argv):
    return subprocess.call(spawn_cmd(gpus, argv))


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the process group has {world} rank(s); "
                         f"launch with torchrun --nproc-per-node {args.gpus}, or without WORLD_SIZE "
                         "(bench.py then spawns the ranks itself)")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: --gpus {world} but only {torch.cuda.device_count()} CUDA device(s)")
    torch.cuda.set_device(local)
    nid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1204_6255_b200.dist import nccl_rendezvous
        _, _, nid = nccl_rendezvous()
        args.mode = "push"                   # the partitioned sweep is push-only
        if args.sched == "block":            # block order is single-GPU; async and bulk shard
            args.sched = "bulk"
    import paper_1204_6255_b200 as di
    if args.mode != "push":
        args.sched = "bulk"
    if args.sched != "block":
        args.blocks = 1
    use_async = args.sched == "async"
    dist_async = use_async and world > 1 and args.dist_async   # F2: ranks meet every 4 cycles
    part = dict(rank=rank, world=world, nccl_id=nid) if world > 1 else dict(build_csc=args.mode != "push")

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    used_spacer = False
    if world > 1:
        # every rank draws only the links of its own source range (equal node ranges; the R-MAT
        # ids are Feistel-relabelled) on its GPU, and uploads them with DI_LOCAL_LINKS: no rank
        # holds the whole link list (C5: 2.16e9 links; ~270e6 per rank at N = 8)
        import digen
        n = digen.CONFIGS[args.config].n
        lo, hi = digen.node_ranges(n, world)[rank]
        t = time.time()
        if digen.CONFIGS[args.config].kind == "rmat":
            s_d, t_d, _ = digen.make_range_gpu(args.config, lo, hi, seed=args.seed, device=dev)
        else:   # host-block recipe: host generator, own sources kept
            src_all, dst_all, _ = digen.make(args.config, seed=args.seed)
            keep = (src_all >= lo) & (src_all < hi)
            s_d = torch.from_numpy(src_all[keep]).to(dev)
            t_d = torch.from_numpy(dst_all[keep]).to(dev)
            del src_all, dst_all, keep
        torch.cuda.synchronize()
        gen_s = time.time() - t
        part["local_range"] = (lo, hi)
        src = dst = None
        L_local = torch.tensor([s_d.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(L_local)
        L = int(L_local.item())
    else:
        src, dst, n, gen_s = make_graph(args.config, args.seed)
        L = len(src)
        # The physical memory behind the graph's arrays changes the solve time by a few per cent
        # (profiles/r2/c5_bench_vs_tool.txt, bench_spacer_ab.txt, placement_sweep.txt): C5 runs in
        # 583-591 ms when the library's pool is carved from memory torch had used and released (links
        # drawn on the GPU, or this spacer) and in 603-624 ms when it follows the 17.3 GB link list
        # in never-used memory; C4 (2.1 GB of links) is 1.2 % faster the plain way. So a link list
        # of more than 4 GiB is preceded by a spacer that is released before the upload;
        # --no-spacer keeps the plain order
        spacer = None
        if not args.no_spacer and 8 * L > (4 << 30):
            spacer = torch.empty(int(torch.cuda.mem_get_info(dev)[0] * 0.5), dtype=torch.uint8, device=dev)
        s_d = torch.from_numpy(src).to(dev)
        t_d = torch.from_numpy(dst).to(dev)
        used_spacer = spacer is not None
        if spacer is not None:
            del spacer
            torch.cuda.empty_cache()

    # ---- a0 build ("Init"), device pointers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = di.Graph(s_d, t_d, n, stream=stream, **part)
    torch.cuda.synchronize()
    init_ms = (time.perf_counter() - t0) * 1e3
    if world > 1:   # the rank's own links, pinned on the host for the e2e steps
        src_p = s_d.cpu().pin_memory()
        dst_p = t_d.cpu().pin_memory()
    del s_d, t_d

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    # headline steps: the solve as one CUDA graph with a device-side while loop (DI_GRAPH_LOOP,
    # single GPU); every timed step is followed, inside the same timed region, by a profiled
    # host-loop solve whose per-kernel CUDA events give the roofline's kernel durations
    use_graph = world == 1

    def one(profile, graph):
        flush.fill_(1)                                   # L2 flush (> 126 MB L2) outside the event pair
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        st = g.solve(d=D, tol=TOL, variant=args.variant, profile=profile, mode=args.mode,
                     blocks=args.blocks, graph_loop=graph, asynchronous=use_async, dist_async=dist_async)
        ev1.record(stream)
        ev1.synchronize()
        assert st["converged"] == 1, st
        return st, ev0.elapsed_time(ev1)

    for _ in range(args.warmup):
        one(False, use_graph)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stats, times, pstats, ptimes = [], [], [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            st, ms = one(False, use_graph)
            stats.append(st)
            times.append(ms)
            st, ms = one(True, False)
            pstats.append(st)
            ptimes.append(ms)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tot_ms = sum(times)
    links = sum(s["link_diffusions"] for s in stats)   # global: the partitioned stats are allreduced
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = links / (tot_ms * 1e-3) / 1e9
    ms_per_step = tot_ms / args.steps

    # ---- roofline of the dominant kernel: algorithmic bytes / event time. DI_ASYNC: k_cycle does
    #      the whole cycle (select + push), so its bytes are the full counted bytes of the cycle;
    #      otherwise k_push's counted push bytes
    peak, peak_src = peaks()
    push_bytes = sum(s["counted_bytes" if use_async else "push_bytes"] for s in pstats) / world
    push_ms = sum(s["push_ms"] for s in pstats)
    push_launches = sum(s["push_launches"] for s in pstats)
    sel_ms = sum(s["select_ms"] for s in pstats)
    ptot_ms = sum(ptimes)
    achieved = push_bytes / (push_ms * 1e-3) / 1e9 if push_ms > 0 else 0.0
    # the instantiation this run's cycles use: the partitioned compact path (N > 1), cold bins
    # (C5 on one GPU: F > 2 x L2), else the plain / warm-tier kernel (profiles/ncu_traffic.json keys)
    # (template arguments LOOPS, DIST, TEST, COLD, WARM; round-1 captures carry the first four)
    keys = ((["k_cycle<0,1,0,1,0>", "k_cycle<0,1,0,1>"] if world > 1 else
             ["k_cycle<0,0,0,1,0>", "k_cycle<0,0,0,1>"] if 8 * n > 2 * 126 * (1 << 20) else ["k_cycle"])
            if use_async else ["k_push"])
    tr = next((v for v in (ncu_traffic(k) for k in keys) if v is not None), None)
    counted = sum(s["counted_bytes"] for s in stats) / world
    kname = ("k_cycle (a2-a6 fused: asynchronous select + push of one cycle)" if use_async else
             "k_push (a5: diffusion of the frontier's fluid)" if args.mode == "push" else
             "k_push + k_pull (a5/a5': diffusion of the frontier's fluid)")
    roofline = {"bound": "hbm", "kernel": kname,
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": tr,
                "frac_vs_8TBps_spec": round(achieved / 8000.0, 4),
                "peak_source": peak_src,
                "bytes_per_launch": push_bytes / max(push_launches, 1),
                "avg_launch_ms": push_ms / max(push_launches, 1),
                "push_share_of_step": round(push_ms / ptot_ms, 4) if ptot_ms else None,
                "select_share_of_step": round(sel_ms / ptot_ms, 4) if ptot_ms else None,
                "measured_on": "profiled host-loop solves interleaved with the timed steps",
                "whole_solve_counted_GBps": round(counted / (tot_ms * 1e-3) / 1e9, 1),
                # the unit that binds the push: scattered fp64 REDs at L2, against the
                # in-L2 ceiling measured by tools/micro/atomics.cu (profiles/micro_atomics.txt)
                # (with the warm tier, part of the link updates are shared-memory adds:
                # this is link updates per second, of which the L2 sees the rest)
                "l2_red": {"achieved_G_per_s": round(sum(s["link_diffusions"] for s in pstats) / world
                                                     / (push_ms * 1e-3) / 1e9, 1) if push_ms > 0 else None,
                           "peak_G_per_s": RED_PEAK, "unit": "G link updates/s (fp64 REDs + warm-tier adds)"}}

    gl_ms = round(statistics.median(ptimes), 3)       # the profiled host-loop solve, for reference
    # warm number (report cold and warm): the same solve without the L2 flush
    warm = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.solve(d=D, tol=TOL, variant=args.variant, mode=args.mode, blocks=args.blocks,
                graph_loop=use_graph, asynchronous=use_async, dist_async=dist_async)
        e1.record(stream)
        e1.synchronize()
        warm.append(e0.elapsed_time(e1))
    warm_ms = round(statistics.median(warm), 3)

    # ---- breadth (outside the timed region): the DI-CYC variant on the same graph,
    #      and the paper's comparators on the GPU at equal accuracy (tol = the DI run's final
    #      normalised error): PI' (push, CSR) and PI (pull, CSC: a second upload)
    variants = None
    if not args.no_breadth:
        variants = {}
        ref = stats[-1]
        cyc = []
        for _ in range(3):
            flush.fill_(1)
            stc = g.solve(d=D, tol=TOL, variant="cyc", mode=args.mode, blocks=args.blocks,
                          graph_loop=use_graph, asynchronous=use_async, dist_async=dist_async)
            cyc.append(stc)
        ms_c = statistics.median(s_["solve_ms"] for s_ in cyc)
        lk_c = cyc[-1]["link_diffusions"]
        variants["DI-CYC"] = {"ms": round(ms_c, 3), "GTEPS": round(lk_c / (ms_c * 1e-3) / 1e9, 3),
                              "sweeps": cyc[-1]["sweeps"], "equivalent_iterations": round(cyc[-1]["equivalent_iterations"], 2),
                              "residual_l1": cyc[-1]["residual_l1"]}
        if world == 1:
            target = ref["error_estimate"]      # the DI run's final sum(F)/(1-d-d e)
            comps = {}
            flush.fill_(1)
            stp = g.solve(d=D, tol=target, variant="pi_push")
            comps["PI'"] = stp
            g_csc = di.Graph(torch.from_numpy(src).to(dev), torch.from_numpy(dst).to(dev), n, stream=stream,
                             build_csc=True)
            flush.fill_(1)
            comps["PI"] = g_csc.solve(d=D, tol=target, variant="pi_pull")
            g_csc.free()
            for k_, st_ in comps.items():
                variants[k_] = {"ms": round(st_["solve_ms"], 3), "iterations": st_["sweeps"],
                                "converged": st_["converged"], "tol": target,
                                "DI_SOP_speedup": round(st_["solve_ms"] / ms_per_step, 2)}

    # ---- e2e through the C ABI with host buffers (H2D of the link list, build, solve, D2H of H)
    if world == 1:
        src_p = torch.from_numpy(src).pin_memory()
        dst_p = torch.from_numpy(dst).pin_memory()
    n_local = g.n_local
    h2d_bytes = 8 * int(src_p.numel())
    H_host = torch.empty(n_local, dtype=torch.float64).pin_memory()
    e2e_ms, e2e_links, e2e_up = [], 0, []
    g.free()
    torch.cuda.empty_cache()
    E2E_WARM = 3                                         # pool growth on the first host-pointer builds
    gc.disable()   # no collector pause of the harness inside a timed step (re-enabled below)
    try:
        if args.build_trace:
            di.set_option("build_trace", 1)
        for k in range(args.e2e_steps + E2E_WARM):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gh = di.Graph(src_p, dst_p, n, stream=stream, **part)  # DI_HOST_PTRS: H2D inside
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st = gh.solve(d=D, tol=TOL, variant=args.variant, mode=args.mode, blocks=args.blocks,
                          asynchronous=use_async, dist_async=dist_async,
                          graph_loop=use_graph)
            t2 = time.perf_counter()
            H = gh.history()
            H_host.copy_(H, non_blocking=True)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            print(f"[bench] e2e step {k}: upload {(t1 - t0) * 1e3:.1f} ms, solve {(t2 - t1) * 1e3:.1f} ms "
                  f"(device {st['solve_ms']:.1f}), H to host {(time.perf_counter() - t2) * 1e3:.1f} ms",
                  file=sys.stderr, flush=True)
            gh.free()
            del H
            if k >= E2E_WARM:
                e2e_ms.append(dt)
                e2e_up.append(round((t1 - t0) * 1e3, 1))
                e2e_links += st["link_diffusions"]
    finally:
        gc.enable()
    e2e_val = e2e_links / (sum(e2e_ms) * 1e-3) / 1e9 if e2e_ms else None
    e2e_serial = e2e_val
    e2e_pipe = None
    if world == 1 and args.e2e_pipeline == 1:
        e2e_pipe = e2e_pipelined(di, src_p, dst_p, n, dev, args, use_async, use_graph)
    elif world == 1 and args.e2e_pipeline == 2:
        e2e_pipe = e2e_copy_overlap(di, src_p, dst_p, n, dev, args, use_async, use_graph)
        if e2e_pipe and e2e_pipe["value"] > e2e_val:
            e2e_val = e2e_pipe["value"]

    # ---- CPU oracle baseline (rank 0, N=1): bounded sample = first cycles of the same solve
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(src, dst, n, args)

    clocks = clk.summary()
    gpu_launches = sum(s["gpu_launches"] for s in stats + pstats)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded R-MAT + repair, digen; stands in for uk-2007-05 / gr0.California)",
        "config": {"workload": f"{args.config}: " + __import__("digen").CONFIGS[args.config].note,
                   "n": n, "links": L, "variant": "DI-" + args.variant.upper(), "d": D,
                   "tol_l1_fluid": TOL, "seed": args.seed, "sweep_mode": args.mode,
                   "schedule": {"async": "asynchronous cycles (DI_ASYNC)",
                                "block": f"block-ordered cycles, K = {args.blocks}",
                                "bulk": "bulk-synchronous sweeps"}[args.sched],
                   "l2": "inputs > 126 MB L2 and 512 MiB L2 flush before each step",
                   "parallelism": (f"1-D node range x{world}, (id, value) lists (peer memory if available)"
                                   + (", asynchronous cycles meeting every 4 (F2)" if dist_async else
                                      ", one exchange per cycle")) if world > 1
                   else "single GPU",
                   "init_build_ms": round(init_ms, 1), "generator_s": round(gen_s, 1),
                   "link_tensors": "allocated above a spacer released before the upload" if used_spacer
                   else "plain allocation order"},
        "time_to_tol_ms": round(ms_per_step, 3),
        "warm_ms_per_step": warm_ms,
        "sweeps": stats[-1]["sweeps"], "equivalent_iterations": round(stats[-1]["equivalent_iterations"], 2),
        "residual_l1": stats[-1]["residual_l1"],
        "hbm_frac_counted_whole_solve": round(counted / (tot_ms * 1e-3) / 1e9 / peak, 4),
        "roofline": roofline,
        "e2e": {"value": round(e2e_val, 3) if e2e_val else None, "unit": UNIT,
                "mode": (("pipelined: a stream of graphs, the H2D copy of step k+1 (copy engine, its own "
                          "stream) overlaps the build (di_graph_upload from device memory), solve and H "
                          "read of step k" if args.e2e_pipeline == 2 else
                          "pipelined: a stream of graphs, the upload of step k+1 (H2D + build, on its own "
                          "stream and host thread) overlaps the solve of step k")
                         if e2e_pipe and e2e_val == e2e_pipe["value"]
                         else "serial: upload, solve, H to host, one graph at a time"),
                "serial": {"value": round(e2e_serial, 3) if e2e_serial else None,
                           "ms_per_step": round(statistics.mean(e2e_ms), 2) if e2e_ms else None,
                           "upload_ms": e2e_up},
                "pipelined": e2e_pipe,
                "ms_per_step": round(statistics.mean(e2e_ms), 2) if e2e_ms else None,
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": 8 * n_local,
                "includes": ("pinned host link list -> di_graph_upload(DI_HOST_PTRS) build -> di_solve -> H to host"
                             + (" (per rank: its own source range, DI_LOCAL_LINKS; bytes per rank)" if world > 1 else ""))},
        "gpu_launches": gpu_launches,
        "host_loop_profiled_ms_per_step": gl_ms,
        "loop": "DI_GRAPH_LOOP (device-side while node)" if use_graph else "host loop",
        "exchange": ({"bytes_per_step_per_gpu": sum(s["exchange_bytes"] for s in stats) / len(stats),
                      "ms_per_step": sum(s["exchange_ms"] for s in stats) / len(stats),
                      "peer_memory_sweeps_per_step": sum(s["p2p_exchanges"] for s in stats) / len(stats),
                      "dense_sweeps_per_step": sum(s["dense_exchanges"] for s in stats) / len(stats),
                      "meetings_per_step": sum(s["meetings"] for s in stats) / len(stats)}
                     if world > 1 else None),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "variants": variants,
        "oracle_time_to_tol": oracle_cached(args.config),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_copy_overlap(di, src_p, dst_p, n, dev, args, use_async, use_graph):
    """End to end over a stream of graphs, the copy engine overlapped: the H2D copy of graph k+1's
    link list from pinned host memory (its own stream, double-buffered device arrays) runs while
    graph k is built from device memory (di_graph_upload with device pointers), solved and its H
    read back to the host; the build and the solve keep the SMs to themselves. Every step's H2D
    copy and D2H read are inside the timed region (steady state: the first step primes the copy);
    value = link diffusions / wall time of the timed steps."""
    import torch
    W, K = 1, args.e2e_steps
    L = int(src_p.numel())
    cs = torch.cuda.Stream(dev)
    ss = torch.cuda.Stream(dev)
    bufs = [(torch.empty(L, dtype=torch.int32, device=dev), torch.empty(L, dtype=torch.int32, device=dev))
            for _ in range(2)]
    evs = [torch.cuda.Event() for _ in range(2)]
    H_host = torch.empty(n, dtype=torch.float64).pin_memory()

    def copy(k):
        b = bufs[k % 2]
        with torch.cuda.stream(cs):
            b[0].copy_(src_p, non_blocking=True)
            b[1].copy_(dst_p, non_blocking=True)
            evs[k % 2].record(cs)

    torch.cuda.synchronize()
    copy(0)
    links, t_first = 0, None
    gc.disable()
    try:
        for k in range(W + K):
            if k == W:
                t_first = time.perf_counter()
            if k + 1 < W + K:
                copy(k + 1)   # into the buffer step k-1 built from (its build is done: synchronised)
            ss.wait_event(evs[k % 2])
            g = di.Graph(bufs[k % 2][0], bufs[k % 2][1], n, stream=ss)
            st = g.solve(d=D, tol=TOL, variant=args.variant, asynchronous=use_async, graph_loop=use_graph)
            with torch.cuda.stream(ss):
                H = g.history()
                H_host.copy_(H, non_blocking=True)
            ss.synchronize()
            assert st["converged"] == 1
            print(f"[bench] copy-overlap step {k}: {(time.perf_counter() - (t_first or time.perf_counter())) * 1e3:.1f} ms "
                  f"(solve device {st['solve_ms']:.1f})", file=sys.stderr, flush=True)
            g.free()
            del H
            if k >= W:
                links += st["link_diffusions"]
    finally:
        gc.enable()
    dt = time.perf_counter() - t_first
    return {"value": round(links / dt / 1e9, 3), "unit": UNIT, "steps": K,
            "ms_per_step": round(dt * 1e3 / K, 2), "graphs_in_flight": 2,
            "overlap": "H2D copy of step k+1 (copy engine) with build + solve + H read of step k",
            "h2d_bytes_per_step": 8 * L, "d2h_bytes_per_step": 8 * n}


def e2e_pipelined(di, src_p, dst_p, n, dev, args, use_async, use_graph):
    """End to end over a stream of graphs through the public API: a host thread uploads graph k+1
    from pinned host memory (di_graph_upload with DI_HOST_PTRS: H2D + build, on its own stream)
    while the main thread solves graph k and reads its H back to the host. Every step's H2D copy
    and D2H read are inside the timed region; value = link diffusions / wall time of all steps."""
    import queue
    import threading
    import torch
    steps = args.e2e_steps + 2
    # the uploads run on low-priority streams: the block scheduler serves the solve's kernels
    # first, the build's kernels fill what the solve leaves, and the copy engine is idle otherwise
    lo_prio, hi_prio = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
        else (0, -1)
    streams = [torch.cuda.Stream(dev, priority=lo_prio) for _ in range(3)]
    solve_streams = [torch.cuda.Stream(dev, priority=hi_prio) for _ in range(3)]
    H_host = torch.empty(n, dtype=torch.float64).pin_memory()
    q = queue.Queue(maxsize=1)
    err = []

    T0 = time.perf_counter()

    def producer():
        try:
            torch.cuda.set_device(dev)
            for k in range(steps):
                s_ = streams[k % 3]
                t_ = (time.perf_counter() - T0) * 1e3
                gk = di.Graph(src_p, dst_p, n, stream=s_)
                print(f"[bench] pipelined upload {k}: {t_:.1f} -> {(time.perf_counter() - T0) * 1e3:.1f} ms",
                      file=sys.stderr, flush=True)
                q.put((k, gk))
        except Exception as e:   # surfaced by the consumer
            err.append(e)
            q.put((None, None))

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = threading.Thread(target=producer, daemon=True)
    th.start()
    links, t_first = 0, None
    for _ in range(steps):
        k, g = q.get()
        if g is None:
            raise err[0]
        t_s = (time.perf_counter() - T0) * 1e3
        g.set_stream(solve_streams[k % 3])   # the solve on a high-priority stream
        with torch.cuda.stream(g.stream):
            # host loop: a new handle's CUDA-graph loop would be captured and instantiated while the
            # other thread's upload runs, which stalled the solve by ~40 ms per step (measured)
            st = g.solve(d=D, tol=TOL, variant=args.variant, asynchronous=use_async, graph_loop=False)
            H = g.history()
            H_host.copy_(H, non_blocking=True)
            g.stream.synchronize()
        assert st["converged"] == 1
        print(f"[bench] pipelined solve {k}: {t_s:.1f} -> {(time.perf_counter() - T0) * 1e3:.1f} ms "
              f"(device {st['solve_ms']:.1f})", file=sys.stderr, flush=True)
        g.free()
        del H
        if k == 1:    # steady state from here: step 0 warms the pool; its upload is not overlapped
            t_first = time.perf_counter()
        elif k > 1:
            links += st["link_diffusions"]
    th.join()
    dt = time.perf_counter() - t_first
    return {"value": round(links / dt / 1e9, 3), "unit": UNIT, "steps": steps - 2,
            "ms_per_step": round(dt * 1e3 / (steps - 2), 2), "graphs_in_flight": 2,
            "h2d_bytes_per_step": 8 * int(src_p.numel()), "d2h_bytes_per_step": 8 * n}


def oracle_cached(config):
    """The sequential oracle's whole solve to ||F||_1 <= 1e-10 on this workload, measured once on a
    GPU box's host core by tools/oracle_time.py and committed (profiles/r2/oracle_<cfg>_full.json);
    the bench's own cpu_baseline times a bounded sample only."""
    path = os.path.join(ROOT, "profiles", "r2", f"oracle_{config}_full.json")
    try:
        with open(path) as f:
            out = json.load(f)
        out["source"] = "cached: " + os.path.relpath(path, ROOT)
        return out
    except Exception:
        return None


def cpu_baseline(src, dst, n, args, budget_cycles=None):
    """Sequential oracle DI-SOP (§2.5.5) on this host, 1 thread, bounded to the first
    `cycles` cycles of the same workload (adjacency build excluded, as the paper's Init)."""
    import oracle
    cycles = budget_cycles or args.cpu_cycles
    prev = os.sched_getaffinity(0)          # pinned to one host core
    core = min(prev)
    os.sched_setaffinity(0, {core})
    try:
        H, F, st = oracle.di(src, dst, n, d=D, tol=TOL, variant=args.variant, max_cycles=cycles)
    finally:
        os.sched_setaffinity(0, prev)
    secs = st["solve_seconds"]
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    return {"value": round(st["diffusions"] / secs / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {st['cycles']} sequential DI-{args.variant.upper()} cycles of {args.config} "
                      f"({st['diffusions']} link diffusions, {secs:.1f} s, loop only)",
            "seconds": round(secs, 2),
            "host": {"cpu": model, "pinned_core": core, "host_cores": os.cpu_count()}}


def launch_check(args):
    """The launch path without a GPU: the same spawn and the same world == --gpus assertion as the
    bench, then one gloo all-gather of the ranks; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the process group has {world} rank(s)")
    if world > 1:
        dist.init_process_group("gloo")
        got = [None] * world
        dist.all_gather_object(got, (rank, os.getpid()))
        dist.destroy_process_group()
    else:
        got = [(0, os.getpid())]
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks": [r for r, _ in got],
                          "pids": len({p for _, p in got})}), flush=True)


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    src, dst, n, _ = make_graph(args.config, args.seed)
    import oracle
    vals, times, last = [], [], None
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(src, dst, n, args)
        if k >= args.warmup:
            vals.append(cb["value"])
            times.append(cb["seconds"] * 1e3)
            last = cb
    value = statistics.mean(vals)
    out = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": max(world, args.gpus),
           "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(statistics.mean(times), 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": f"{args.config}: " + __import__("digen").CONFIGS[args.config].note,
                      "variant": "DI-" + args.variant.upper(), "d": D, "tol_l1_fluid": TOL},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": last["sample"], "host": last.get("host")},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--variant", default="sop", choices=["sop", "cyc"])
    ap.add_argument("--mode", default="push", choices=["push", "pull", "auto"])
    ap.add_argument("--sched", default="async", choices=["async", "block", "bulk"],
                    help="async: one persistent kernel per cycle (DI_ASYNC); block: K ordered blocks "
                         "per cycle (DI_BLOCKS); bulk: bulk-synchronous sweeps")
    ap.add_argument("--blocks", type=int, default=8, help="K for --sched block")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--dist-async", action="store_true",
                    help="N > 1: asynchronous multi-GPU cycles (DI_DIST_ASYNC, SURVEY F2)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-cycles", type=int, default=12)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-spacer", action="store_true",
                    help="one GPU, link lists over 4 GiB: no spacer below the link tensors (see run_ours)")
    ap.add_argument("--no-breadth", action="store_true", help="skip the DI-CYC / PI / PI' rows")
    ap.add_argument("--e2e-pipeline", type=int, default=0, choices=(0, 1, 2),
                    help="also measure e2e over a stream of graphs: 1 = the upload of k+1 (host link "
                         "list: H2D + build) overlaps the solve of k; 2 = only the H2D copy of k+1 "
                         "overlaps the build and solve of k (device-pointer upload)")
    ap.add_argument("--build-trace", action="store_true",
                    help="diagnostic: the library's build_trace option during the e2e uploads (stderr)")
    ap.add_argument("--launch-check", action="store_true",
                    help="only check the launch: N ranks over gloo (CPU), world == --gpus, rank 0 prints "
                         "one JSON line (tests/test_bench_launch.py)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch this command under torch.distributed.run (rendezvous on
        # 127.0.0.1); rank 0 prints the JSON line, the exit code is the launcher's
        sys.exit(spawn(args.gpus, sys.argv[1:]))
    if args.launch_check:
        return launch_check(args)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
