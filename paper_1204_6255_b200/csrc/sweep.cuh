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
  double *partials;     // 4 per select tile: q, s, e, taken
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
  // block-ordered sweeps (F1): this launch scans select tiles [t0, t1), sub-sweep blk
  // of `blocks` per cycle (blocks = 1: the plain bulk sweep over every tile)
  int64_t t0, t1;
  int blk, blocks;
  double *ppartials;    // 8 per finaliser slice: q, s, e, taken, sel, nd, links, 0
  int hot_shift;        // replicated hot accumulators: number of hot ids, -1 = off (every
                        // single-GPU push schedule and PI' use them; top share > kReplShare = 0.05 %)
  double *rep;
  const int64_t *hub;   // DI_ASYNC hub items (async.cu), n_hub of them
  int n_hub;
  unsigned long long *times;  // option cycle_times diagnostic (async.cu), nullptr = off
  double *rec_T, *rec_v;      // di_test_cycle records (async.cu, TEST instantiation only)
  // cold bins (async.cu COLD instantiation): targets j >= cold_lo become records of bin
  // (j - cold_lo) >> cold_shift in region cold_off[b] of the arena
  int64_t cold_lo;
  int64_t cold_hot_tiles;   // tiles holding first-tier ids (interleaved over the cycle)
  int cold_shift, cold_nbins;
  int long_lanes;           // k_cycle long rows: lane-consecutive targets (option long_lanes)
  int64_t claim_lo, claim_hi;   // k_cycle: claims [claim_lo, claim_hi) (claim_hi < 0: all)
  int warm;                 // k_cycle warm tier: warm-rank slots in shared memory (0: off), the
  int warm_hot, warm_shift; //   ids warm_hot + k << warm_shift (k < warm), and the hot ids
  int warm_flush;           //   flushed every warm_flush tiles of a CTA too (0: at its end only)
  ColdRec *cold_rec;
  const int64_t *cold_off;
  unsigned long long *cold_top;
  int32_t *cold_fill;
};

// What one sweep moved: r_{n+1} = q + s (a2), dangling absorption e, counters.
struct SweepSums {
  double q, s, e, taken;
  int64_t sel, nd, lk, scanned;
};

// Two-level fixed-order reduction of the per-tile partials written by k_select (a2).
// Level 1: slice p of P (every block of the push/pull grid reduces a fixed contiguous slice of
// the tiles [t0, t1) into ppartials[p]). Level 2 (reduce_partials): the last block reduces the
// P slice results. Both orders are fixed, so the sums are reproducible for a given grid.
__device__ __forceinline__ void slice_partials(const SweepArgs &a, int p, int P, int nthreads) {
  __shared__ double s_sl[32][4];
  __shared__ long long s_isl[32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nt = a.t1 - a.t0;
  const int64_t b0 = a.t0 + nt * p / P, b1 = a.t0 + nt * (p + 1) / P;
  double aq = 0.0, as = 0.0, ae = 0.0, at = 0.0;
  long long c_sel = 0, c_nd = 0, c_lk = 0;
  for (int64_t tt = b0 + threadIdx.x; tt < b1; tt += nthreads) {
    const double2 x01 = __ldcg(reinterpret_cast<const double2 *>(a.partials) + 2 * tt);
    const double2 x23 = __ldcg(reinterpret_cast<const double2 *>(a.partials) + 2 * tt + 1);
    const longlong2 c01 = __ldcg(reinterpret_cast<const longlong2 *>(a.ipartials) + 2 * tt);
    const longlong2 c23 = __ldcg(reinterpret_cast<const longlong2 *>(a.ipartials) + 2 * tt + 1);
    aq += x01.x;
    as += x01.y;
    ae += x23.x;
    at += x23.y;
    c_sel += c01.x;
    c_nd += c01.y;
    c_lk += c23.x;
  }
  aq = warp_sum(aq);
  as = warp_sum(as);
  ae = warp_sum(ae);
  at = warp_sum(at);
  c_sel = warp_sum(c_sel);
  c_nd = warp_sum(c_nd);
  c_lk = warp_sum(c_lk);
  if (lane == 0) {
    s_sl[warp][0] = aq;
    s_sl[warp][1] = as;
    s_sl[warp][2] = ae;
    s_sl[warp][3] = at;
    s_isl[warp][0] = c_sel;
    s_isl[warp][1] = c_nd;
    s_isl[warp][2] = c_lk;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[4] = {0.0, 0.0, 0.0, 0.0};
    long long c[3] = {0, 0, 0};
    for (int w = 0; w < nthreads / 32; w++) {
      for (int k = 0; k < 4; k++) r[k] += s_sl[w][k];
      for (int k = 0; k < 3; k++) c[k] += s_isl[w][k];
    }
    double *o = a.ppartials + 8 * (int64_t)p;
    reinterpret_cast<double2 *>(o)[0] = make_double2(r[0], r[1]);
    reinterpret_cast<double2 *>(o)[1] = make_double2(r[2], r[3]);
    reinterpret_cast<longlong2 *>(o)[2] = make_longlong2(c[0], c[1]);
    reinterpret_cast<longlong2 *>(o)[3] = make_longlong2(c[2], 0);
  }
}

// Level 2: reduce the P slice results (valid in thread 0). Called by one whole block after
// every slice has been written.
__device__ __forceinline__ SweepSums reduce_partials(const SweepArgs &a, int P, int nthreads) {
  __shared__ double s_fin[32][4];
  __shared__ long long s_ifin[32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double aq = 0.0, as = 0.0, ae = 0.0, at = 0.0;
  long long c_sel = 0, c_nd = 0, c_lk = 0;
  for (int p = threadIdx.x; p < P; p += nthreads) {
    const double *o = a.ppartials + 8 * (int64_t)p;
    const double2 x01 = __ldcg(reinterpret_cast<const double2 *>(o));
    const double2 x23 = __ldcg(reinterpret_cast<const double2 *>(o) + 1);
    const longlong2 c01 = __ldcg(reinterpret_cast<const longlong2 *>(o) + 2);
    const longlong2 c23 = __ldcg(reinterpret_cast<const longlong2 *>(o) + 3);
    aq += x01.x;
    as += x01.y;
    ae += x23.x;
    at += x23.y;
    c_sel += c01.x;
    c_nd += c01.y;
    c_lk += c23.x;
  }
  aq = warp_sum(aq);
  as = warp_sum(as);
  ae = warp_sum(ae);
  at = warp_sum(at);
  c_sel = warp_sum(c_sel);
  c_nd = warp_sum(c_nd);
  c_lk = warp_sum(c_lk);
  if (lane == 0) {
    s_fin[warp][0] = aq;
    s_fin[warp][1] = as;
    s_fin[warp][2] = ae;
    s_fin[warp][3] = at;
    s_ifin[warp][0] = c_sel;
    s_ifin[warp][1] = c_nd;
    s_ifin[warp][2] = c_lk;
  }
  __syncthreads();
  const int64_t n0 = a.t0 * kSelTile, n1 = a.t1 * kSelTile < a.n ? a.t1 * kSelTile : a.n;
  SweepSums r{0.0, 0.0, 0.0, 0.0, 0, 0, 0, n1 - n0};
  if (threadIdx.x == 0) {
    for (int w = 0; w < nthreads / 32; w++) {
      r.q += s_fin[w][0];
      r.s += s_fin[w][1];
      r.e += s_fin[w][2];
      r.taken += s_fin[w][3];
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
  if (a.blocks > 1) {  // sub-sweep blk of a block-ordered cycle (F1)
    const bool first = a.blk == 0, last = a.blk == a.blocks - 1;
    const double d = vs->d;
    const int variant = vs->variant;
    // running sum F: r (cycle start) - fluid taken from F + fluid pushed (every sub-sweep)
    const double r_run = __dadd_rn(__dsub_rn(first ? vs->r : vs->r_run, x.taken), x.s);
    const double e_tot = vs->e + x.e;
    const int64_t sel_c = (first ? 0 : vs->sel_cyc) + x.sel;
    const int64_t lk_c = (first ? 0 : vs->links_cyc) + x.lk;
    vs->r_run = r_run;
    vs->sel_cyc = sel_c;
    vs->links_cyc = lk_c;
    vs->e = e_tot;
    vs->q = x.q;
    vs->s = x.s;
    vs->e_sw = x.e;
    vs->selected_total = vs->selected_total + x.sel;
    vs->selected_nd_total = vs->selected_nd_total + x.nd;
    vs->links_total = vs->links_total + x.lk;
    vs->scanned_total = vs->scanned_total + x.scanned;
    const double err = vs->paper_err ? r_run / (1.0 - d - d * e_tot) : r_run;
    const int stop = err <= vs->tol;  // checked after every sub-sweep (r_run is sum F)
    vs->stop = stop;
    if (last || stop) {
      const int64_t sw = vs->sweeps;
      if (vs->trace && sw < kLogCap) {
        a.log_r[sw] = vs->r;
        a.log_sel[sw] = sel_c;
        a.log_links[sw] = lk_c;
        a.log_mode[sw] = 0;
      }
      if (vs->guard && variant != DI_CYC) vs->guards = vs->guards + 1;
      vs->sweeps = sw + 1;
      vs->r = r_run;  // threshold fluid of the next cycle (once per cycle)
      vs->guard = (sel_c == 0 && !stop && variant == DI_SOP) ? 1 : 0;
    }
    for (int b = 0; b < kBins; b++) {
      vs->bin_count[b] = (int64_t)vs->bin_fill[b][0];
      vs->bin_fill[b][0] = 0;
    }
    vs->ticket = 0;
    return;
  }
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

// the replicated hot accumulators into F, cleared (every push kernel's last block, all threads)
__device__ __forceinline__ void fold_replicas(const SweepArgs &a, int nthreads) {
  if (a.hot_shift <= 0 || !a.rep) return;
  for (int k = threadIdx.x; k < a.hot_shift; k += nthreads) {
    double acc = 0.0;
    for (int c = 0; c < kRepCopies; c++) {
      double *p = a.rep + (int64_t)(c * kHotRanks + k) * kRepStride;
      acc += __ldcg(p);
      *p = 0.0;
    }
    if (acc != 0.0) a.F[k] += acc;
  }
}

__device__ __forceinline__ void finalize_sweep(const SweepArgs &a, int P, int nthreads) {
  fold_replicas(a, nthreads);
  const SweepSums x = reduce_partials(a, P, nthreads);
  if (threadIdx.x == 0) apply_sweep(a, x);
}

// Column ids are read as aligned int4 groups (one LSU instruction per 4 links); elements of a
// group outside [beg, end) are masked. The col array carries 8 elements of tail padding.
// Each valid target j != i receives v with a fire-and-forget RED.
// Hot ids j < hot_lim (replicated accumulators; 0 when off) go to copy `copy` of j.
template <bool LOOPS>
__device__ __forceinline__ void red_group(double *__restrict__ F, double *__restrict__ rep,
                                          int32_t hot_lim, int copy, int4 x, int64_t p0,
                                          int64_t beg, int64_t end, int32_t gi, double v,
                                          uint64_t fpol) {
  const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end && (!LOOPS || jj[c] != gi)) {
      if (jj[c] < hot_lim)
        red_add_f64(rep + (int64_t)(copy * kHotRanks + jj[c]) * kRepStride, v);
      else
        red_add_f64_hint(F + jj[c], v, fpol);
    }
  }
}

// blk / blocks: sub-sweep blk of `blocks` block-ordered sub-sweeps (tile range [t0, t1))
// Multi-GPU sweep state (dist.cu, async.cu): remote accumulator, send records, sweep header.
struct DistArgs {
  double *R;
  double *sval;
  unsigned long long *tcnt;  // [(world + 1) * 32]: records per owner, one line each; a ticket
  int64_t *sendcnt;          // [world] (view into the sweep header)
  double *dsum;              // q, s, e, taken
  int64_t *isum;             // sel, nd, lk, scanned
  DistBounds bd;
  int rank;
  // fused exchange (dist.cu): records go straight into the owner's inbox through peer memory;
  // inbox[p] = rank p's inbox as mapped here, segment (parity, source) of icap records
  char *inbox[kMaxWorld];
  int64_t icap;
  int ipar;    // cycle parity: double-buffered segments (a rank is at most one cycle ahead)
  int p2p;     // 1: k_compact_remote writes into inbox[p]; 0: into sval (then exchange())
  int ring;    // DI_DIST_ASYNC: append at the ring tail, publish it, sum the sent fluid
  unsigned long long *tsent;  // [kMaxWorld] records sent to each owner so far (ring tails)
  double *sent;               // fluid compacted this cycle (ring mode)
  // compact remote path: the first rt[p] ids of every range p are its hot remote
  // targets, accumulated in racc[hoff[p] + (j - b[p])] (L2-resident); a push to a colder remote
  // target is a 16-B record written straight into the owner's inbox (cold region of this
  // sender, parity ipar), in warp chunks reserved with the counters ctop[2p + parity]
  int compact;                // 1: this path (k_cycle<DIST, COLD>, k_compact_remote over racc)
  double *racc;
  int64_t rt[kMaxWorld];
  int64_t hoff[kMaxWorld + 1];
  int64_t ccap;               // cold records per (sender, parity) region of an inbox
  int64_t cwin;               // cold targets encoded n + sum(rt) + p * cwin + (j - b[p])
  size_t cold_off0, fill_off0;  // byte offsets of the cold regions / their chunk fills in an inbox
  unsigned long long *ctop;   // [2 * kMaxWorld] one line each
  int64_t *coldcnt;           // [world] (view into the sweep header, after sendcnt)
};

inline DistArgs dist_args(Graph &g) {
  DistArgs x;
  for (int p = 0; p < kMaxWorld; p++) x.inbox[p] = (p < (int)g.inbox.size()) ? g.inbox[p] : nullptr;
  x.icap = g.icap;
  x.ipar = 0;
  x.p2p = 0;
  x.ring = 0;
  x.tsent = g.ring;
  x.sent = g.ring ? reinterpret_cast<double *>(g.ring + 3 * kMaxWorld) : nullptr;
  x.R = g.R;
  x.sval = g.sval;
  x.tcnt = g.tcnt;
  x.sendcnt = g.sendcnt;
  x.dsum = g.dsum;
  x.isum = g.isum;
  x.bd = g.bounds;
  x.rank = g.rank;
  x.compact = 0;
  x.racc = g.racc;
  x.hoff[0] = 0;
  for (int p = 0; p < kMaxWorld; p++) {
    x.rt[p] = p < g.world ? g.rtier[p] : 0;
    x.hoff[p + 1] = x.hoff[p] + x.rt[p];
  }
  x.ccap = g.ccap;
  x.cwin = g.cwin;
  x.cold_off0 = g.cold_off0;
  x.fill_off0 = g.fill_off0;
  x.ctop = g.ctop;
  x.coldcnt = g.sendcnt ? g.sendcnt + g.world : nullptr;
  return x;
}

// sweep header words per rank: 8 sums, then per peer the compact records and the cold records
// sent to it; global_sum_F's scratch follows the header
__host__ __device__ inline int hdr_words(int world) { return 8 + 2 * world; }


// A push to a target j that another rank owns: an fp64 RED into the remote accumulator R[j]
// (fire-and-forget like the local push). The touched entries are found afterwards by one
// compaction scan over R (k_compact_remote, dist.cu): 8 B per remote node per sweep instead of an
// atomic with return per remote link (C4 at G = 8: ~15M remote nodes vs ~200M remote links).
__device__ __forceinline__ void push_remote(const DistArgs &x, int32_t j, double v) {
  red_add_f64(x.R + j, v);
}

inline SweepArgs sweep_args(Graph &g, int test_mode, int blk = 0, int blocks = 1) {
  SweepArgs a;
  const int64_t nt = select_tiles(g.n);
  a.t0 = nt * blk / blocks;
  a.t1 = nt * (blk + 1) / blocks;
  a.blk = blk;
  a.blocks = blocks;
  a.ppartials = g.ppartials;
  // replicated hot accumulators (one GPU, hot placement on, allocated by prepare_cycle)
  a.hot_shift = (g.rep && g.reordered && g.hot_acc && !g.partitioned && g.hot_count > 0)
                    ? (int)g.hot_count
                    : -1;
  a.rep = g.rep;
  a.hub = nullptr;
  a.n_hub = 0;
  a.times = nullptr;
  a.rec_T = nullptr;
  a.rec_v = nullptr;
  a.cold_lo = INT64_MAX;
  a.cold_hot_tiles = 0;
  a.long_lanes = 0;
  a.warm = 0;
  a.claim_lo = 0;
  a.claim_hi = -1;
  a.warm_hot = 0;
  a.warm_shift = 0;
  a.warm_flush = 0;
  a.cold_shift = 0;
  a.cold_nbins = 0;
  a.cold_rec = nullptr;
  a.cold_off = nullptr;
  a.cold_top = nullptr;
  a.cold_fill = nullptr;
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
