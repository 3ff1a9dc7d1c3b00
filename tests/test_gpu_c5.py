"""C5 (BASELINE configs[4], the north_star workload: R-MAT N = 2^27, L ~ 2.16e9) at full size, in the
launch configurations bench.py times with --config c5: one GPU (asynchronous cycles in the
device-side graph loop; cold bins on by the auto rule, F = 1 GB >> L2) and 8 partitioned ranks
(the compact remote path through peer memory, here 8 emulated ranks sharing this GPU, every rank
drawing only its own source range as bench.py --gpus 8 does).

The sequential oracle needs ~390 s for C5 (profiles/r2/c5_oracle_parity_final.txt holds that gate:
9.9e-11), so this test checks what holds at any size:
  - ||F||_1 <= 1e-10 at the stop (P:282 with the absolute target of north_star), F >= 0, H >= 0;
  - the invariant F = B + P.H - H on 2000 sampled nodes, to the rounding bound of the
    running sums that built F and H (k_in pushes and one take per cycle; _sampled_invariant);
  - conservation sum F + (1-d) sum_{out>0} H + sum_{out=0} H = sum B = 1 - d (every diffusion moves
    fluid, dangling nodes absorb it: P:264-274);
  - the 8-rank solve against the 1-GPU solve: both stop at ||F||_1 <= 1e-10, so each is within
    1e-10/(1-d) of X and they are within 2e-10/(1-d) of each other (||X - H||_1 <= ||F||_1/(1-d)).
The sampled in-link sums are computed with plain torch ops on the generator's link list (test-side
plumbing, not the library)."""
import threading

import numpy as np
import pytest

import digen
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
D, TOL = 0.85, 1e-10
EPS = 2.0 ** -53


def _sampled_invariant(torch, s, t, n, H, F, sample, cycles):
    """max over sampled i of |F_i - (B_i + sum_{j->i} d H_j/out_j - H_i)| / rounding bound. F_i is a
    running fp64 sum of every push to i and every take from it (at most k_in pushes and one take per
    cycle), H_j a sum of its takes (one per cycle), each push d*T/o two roundings, the test's sum k_in
    more: each operation errs by at most eps times the magnitude it touches, <= B_i + ph_i + H_i."""
    smp = torch.from_numpy(sample).to(s.device)
    flag = torch.zeros(n, dtype=torch.bool, device=s.device)
    flag[smp] = True
    out = torch.zeros(n, dtype=torch.float64, device=s.device)
    si, ti = [], []
    for a, b in zip(s.split(1 << 28), t.split(1 << 28)):   # chunks: int64 temporaries stay small
        out += torch.bincount(a.long(), minlength=n).double()
        m = flag[b.long()]
        si.append(a[m].long())
        ti.append(b[m].long())
    si, ti = torch.cat(si), torch.cat(ti)
    del flag
    ph = torch.zeros(n, dtype=torch.float64, device=s.device)
    ph.index_add_(0, ti, D * H[si] / out[si])
    kin = torch.bincount(ti, minlength=n).double()
    resid = (1 - D) / n + ph[smp] - H[smp]
    k = kin[smp]
    bound = ((k + 2) * cycles + k + 4) * EPS * ((1 - D) / n + ph[smp] + H[smp] + F[smp])
    return float(((resid - F[smp]).abs() / bound).max()), out


def test_c5_full_size_one_gpu_and_8_ranks():
    need_gpu()
    import torch
    import paper_1204_6255_b200 as di
    from paper_1204_6255_b200.dist import assemble, run_local_group
    n = digen.CONFIGS["c5"].n
    assert n == 1 << 27
    s, t, _ = digen.make_range_gpu("c5", 0, n)
    L = s.numel()
    assert 2.0e9 < L < 2.3e9
    g = di.Graph(s, t, n)
    st = g.solve(d=D, tol=TOL, asynchronous=True, graph_loop=True)
    assert st["converged"] == 1 and st["residual_l1"] <= TOL, st
    H1 = g.history()
    _, F = g.residual(return_F=True)
    assert float(F.min()) >= 0.0 and float(H1.min()) >= 0.0
    assert abs(float(F.sum()) - st["residual_l1"]) <= 1e-12 * st["residual_l1"] + 1e-22
    sample = np.random.default_rng(5).choice(n, 2000, replace=False)
    worst, out = _sampled_invariant(torch, s, t, n, H1, F, sample, st["sweeps"])
    assert worst <= 1.0, worst
    cons = float(F.sum()) + (1 - D) * float(H1[out > 0].sum()) + float(H1[out == 0].sum())
    assert abs(cons - (1 - D)) <= 1e-12, cons
    print(f"\nC5 1 GPU: {st['sweeps']} cycles, {st['equivalent_iterations']:.2f} eq-iter, ||F||_1 = "
          f"{st['residual_l1']:.3e}, invariant max/bound = {worst:.3f}, conservation error {cons - (1 - D):.2e}")
    H1 = H1.cpu().numpy()
    del s, t, F, out
    g.free()
    torch.cuda.empty_cache()

    G = 8
    ranges = digen.node_ranges(n, G)
    gen = threading.Lock()

    def rank(r, grp):
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            lo, hi = ranges[r]
            with gen:   # one rank's generator at a time, its cache handed back before the uploads
                sr, tr, _ = digen.make_range_gpu("c5", lo, hi)
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
            gr = di.Graph(sr, tr, n, rank=r, world=G, group=grp, stream=stream, local_range=(lo, hi))
            del sr, tr
            st_ = gr.solve(d=D, tol=TOL, asynchronous=True)
            out_ = ((gr.lo, gr.hi), gr.history().cpu().numpy(), st_, gr.n_links)
            gr.free()
        return out_

    res = run_local_group(G, rank, timeout=1800)
    assert sum(x[3] for x in res) == L          # the ranks' own links tile the graph
    for x in res:
        assert x[2]["converged"] == 1 and x[2]["residual_l1"] <= TOL
    H8 = assemble([x[1] for x in res], [x[0] for x in res], n)
    diff = float(np.abs(H8 - H1).sum())
    print(f"C5 8 ranks: {res[0][2]['sweeps']} cycles, {res[0][2]['equivalent_iterations']:.2f} eq-iter, "
          f"||H_8 - H_1||_1 = {diff:.3e} (bound {2 * TOL / (1 - D):.3e})")
    assert diff <= 2 * TOL / (1 - D), diff
