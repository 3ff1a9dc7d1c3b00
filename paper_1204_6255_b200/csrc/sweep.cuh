// sweep.cuh — the per-sweep argument block and the sweep finaliser,
// shared by the single-GPU kernels (diffusion.cu) and the partitioned ones (dist.cu).
#pragma once
#include "di_common.cuh"
#include "kern_util.cuh"

namespace di {

struct SweepArgs {
  double *F, *H;
  const int32_t *deg, *kloop;
  const int64_t *row_ptr;
  const int32_t *col;
  int64_t n;            // owned nodes
  int64_t lo;           // global id of local node 0
  int64_t ntiles;
  double L_total;       // global link count (threshold r/L)
  Scalars *sc;
  Frontier fr;
  double *partials;     // 3 per select tile
  int64_t *ipartials;   // 4 per select tile
  double *log_r;
  int64_t *log_sel, *log_links;
  uint8_t *log_mode;
  int test_mode;
  int red_hint;         // 1: REDs into F carry an L2 evict_last policy
  double *S;            // pull variant: dense sent value per node (0 if not diffused)
  const int32_t *csc_row;
  PullEntry *pe[kPullBins];
  int64_t pe_count[kPullBins];
};

// What one sweep moved: r_{n+1} = q + s (a2), dangling absorption e, counters.
struct SweepSums {
  double q, s, e;
  int64_t sel, nd, lk, scanned;
};

// Fixed-order reduction of the per-tile partials written by k_select. Called by one whole
// block after every select tile has finished; the result is valid in thread 0.
__device__ __forceinline__ SweepSums reduce_partials(const SweepArgs &a, int nthreads) {
  __shared__ double s_fin[32][3];
  __shared__ long long s_ifin[32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double aq = 0.0, as = 0.0, ae = 0.0;
  long long c_sel = 0, c_nd = 0, c_lk = 0;
#pragma unroll 4
  for (int64_t tt = threadIdx.x; tt < a.ntiles; tt += nthreads) {
    aq += __ldcg(a.partials + tt * 3 + 0);
    as += __ldcg(a.partials + tt * 3 + 1);
    ae += __ldcg(a.partials + tt * 3 + 2);
    const longlong2 c01 = __ldcg(reinterpret_cast<const longlong2 *>(a.ipartials) + 2 * tt);
    const longlong2 c23 = __ldcg(reinterpret_cast<const longlong2 *>(a.ipartials) + 2 * tt + 1);
    c_sel += c01.x;
    c_nd += c01.y;
    c_lk += c23.x;
  }
  aq = warp_sum(aq);
  as = warp_sum(as);
  ae = warp_sum(ae);
  c_sel = warp_sum(c_sel);
  c_nd = warp_sum(c_nd);
  c_lk = warp_sum(c_lk);
  if (lane == 0) {
    s_fin[warp][0] = aq;
    s_fin[warp][1] = as;
    s_fin[warp][2] = ae;
    s_ifin[warp][0] = c_sel;
    s_ifin[warp][1] = c_nd;
    s_ifin[warp][2] = c_lk;
  }
  __syncthreads();
  SweepSums r{0.0, 0.0, 0.0, 0, 0, 0, a.n};
  if (threadIdx.x == 0) {
    for (int w = 0; w < nthreads / 32; w++) {
      r.q += s_fin[w][0];
      r.s += s_fin[w][1];
      r.e += s_fin[w][2];
      r.sel += s_ifin[w][0];
      r.nd += s_ifin[w][1];
      r.lk += s_ifin[w][2];
    }
  }
  return r;
}

// The sweep's effect on the loop state (thread 0 only): r_{n+1}, e, the stop test (P:256,
// P:278-283), the starvation guard (reading G5), counters, the trace, bin counts.
__device__ __forceinline__ void apply_sweep(const SweepArgs &a, const SweepSums &x) {
  volatile Scalars *vs = a.sc;
  const int64_t sw = vs->sweeps;
  const double d = vs->d, r = vs->r;
  const int variant = vs->variant;
  const bool guarded = vs->guard && variant != DI_CYC;
  const int mode = vs->mode;
  const bool pulled = mode == MODE_PULL || (mode == MODE_AUTO && x.lk > vs->pull_thr);
  if (vs->trace && sw < kLogCap) {
    a.log_r[sw] = r;
    a.log_sel[sw] = x.sel;
    a.log_links[sw] = x.lk;
    a.log_mode[sw] = pulled ? 1 : 0;
  }
  if (pulled) vs->pull_sweeps = vs->pull_sweeps + 1;
  vs->fill_links[0] = 0;
  const double r_next = x.q + x.s;  // r_{n+1} = q_n + s_n (a2)
  const double e_tot = vs->e + x.e;
  vs->e = e_tot;
  vs->q = x.q;
  vs->s = x.s;
  vs->e_sw = x.e;
  vs->r = r_next;
  vs->sweeps = sw + 1;
  vs->selected_total = vs->selected_total + x.sel;
  vs->selected_nd_total = vs->selected_nd_total + x.nd;
  vs->links_total = vs->links_total + x.lk;
  vs->scanned_total = vs->scanned_total + x.scanned;
  if (guarded) vs->guards = vs->guards + 1;
  const double err = vs->paper_err ? r_next / (1.0 - d - d * e_tot) : r_next;
  const int stop = err <= vs->tol;
  vs->stop = stop;
  vs->guard = (x.sel == 0 && !stop && variant == DI_SOP) ? 1 : 0;
  for (int b = 0; b < kBins; b++) {
    vs->bin_count[b] = (int64_t)vs->bin_fill[b][0];
    vs->bin_fill[b][0] = 0;
  }
  vs->ticket = 0;
}

__device__ __forceinline__ void finalize_sweep(const SweepArgs &a, int nthreads) {
  const SweepSums x = reduce_partials(a, nthreads);
  if (threadIdx.x == 0) apply_sweep(a, x);
}

// Column ids are read as aligned int4 groups (one LSU instruction per 4 links); elements of a
// group outside [beg, end) are masked. The col array carries 8 elements of tail padding.
// Each valid target j != i receives v with a fire-and-forget RED.
template <bool LOOPS>
__device__ __forceinline__ void red_group(double *__restrict__ F, int4 x, int64_t p0, int64_t beg,
                                          int64_t end, int32_t gi, double v, uint64_t fpol) {
  const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end && (!LOOPS || jj[c] != gi)) red_add_f64_hint(F + jj[c], v, fpol);
  }
}

inline SweepArgs sweep_args(Graph &g, int test_mode) {
  SweepArgs a;
  a.F = g.F;
  a.H = g.H;
  a.deg = g.deg;
  a.kloop = g.kloop;
  a.row_ptr = g.row_ptr;
  a.col = g.col;
  a.n = g.n;
  a.lo = g.lo;
  a.ntiles = select_tiles(g.n);
  a.L_total = (double)g.l_global;
  a.sc = g.sc;
  a.fr = g.fr;
  a.partials = g.partials;
  a.ipartials = g.ipartials;
  a.log_r = g.log_r;
  a.log_sel = g.log_sel;
  a.log_links = g.log_links;
  a.log_mode = g.log_mode;
  a.test_mode = test_mode;
  a.red_hint = g.red_hint;
  a.S = g.S;
  a.csc_row = g.csc_row;
  for (int b = 0; b < kPullBins; b++) {
    a.pe[b] = g.pe[b];
    a.pe_count[b] = g.pe_count[b];
  }
  return a;
}

}  // namespace di
