// async.cu — asynchronous D-iteration cycles: one persistent kernel per cycle (DI_ASYNC).
//
// The paper's cycle visits the nodes in order and reads the LIVE fluid: fluid that
// node i pushes to a later node j is diffused by j in the same cycle. Bulk sweeps (R1) lose that
// (fluid waits for the next sweep); block-ordered cycles (R5) recover part of it at the price of
// 2K kernel boundaries per cycle. Here one persistent grid runs the whole cycle:
//   - CTAs take tiles of kCycTile (512) consecutive nodes in increasing order from a global
//     counter (hub items of the hottest rows are claimed right after tile 0, see below);
//   - a node is selected against the cycle's threshold t = r/L (r once per cycle) and
//     the fluid f the test read is TAKEN with a RED F_i -= f, so fluid that other CTAs push into
//     F_i concurrently is never lost: it stays in F_i for the next visit (any diffusion
//     order keeps F = B + P.H - H); (round 1 took it with an atomic exchange F_i <- 0, which the
//     record mode of di_test_cycle still uses);
//   - the CTA pushes the tile's rows immediately from shared-memory lists: rows of <= 16 links
//     a lane each (32 per warp claim), 17-256 links by 8-lane groups (front of the row list),
//     longer rows as 1024-link chunks claimed by the CTA's warps (back of the row list).
// The order of diffusions is the dynamic order of the tiles, so iterates are not reproducible
// bit for bit (like every fp64-atomic push); the fixed point and the tolerance are those of the
// paper's method. The last CTA reduces the per-CTA sums, applies r_{c+1} = r_c - taken + pushed,
// the stop test and the starvation guard (reading G5), and rewinds the tile counter.
#include <algorithm>
#include <vector>

#include "sweep.cuh"

namespace di {
namespace {

#ifndef DI_ASYNC_THREADS
#define DI_ASYNC_THREADS 256
#endif
constexpr int kAsyncThreads = DI_ASYNC_THREADS;
#ifndef DI_CYC_ITEMS
#define DI_CYC_ITEMS 2
#endif
constexpr int kCycItems = DI_CYC_ITEMS;               // consecutive nodes per thread (1 or even)
constexpr int kCycTile = kAsyncThreads * kCycItems;   // nodes per tile
#ifndef DI_ASYNC_SMALL
#define DI_ASYNC_SMALL 16
#endif
#ifndef DI_ASYNC_MID
#define DI_ASYNC_MID 256
#endif
#ifndef DI_ASYNC_CHUNK
#define DI_ASYNC_CHUNK 1024
#endif
// The window of nodes in flight (CTAs x tile) sets how close the order is to the paper's
// sequential cycle: 1024-node tiles x 4 CTAs/SM: C4 43 cycles / 60.2 ms, C2 3.6 ms; 3 CTAs/SM:
// 42 / 58.7 ms, C2 3.2 ms; 512-node tiles (2 nodes per thread) x 4 CTAs/SM: C4 42 / 58.2 ms,
// C3 25.8 -> 24.2 ms, C2 3.0 ms at the same per-link rate (tools/exp/async.py)
#ifndef DI_TAKE_SUB
#define DI_TAKE_SUB 1   // a selected node's fluid taken as F_i -= f (a RED) (0: an atomic exchange;
                        // C4 52.8 -> 52.7 ms, C3 23.6 -> 22.9 ms: no round trip to wait for)
#endif
#ifndef DI_LL_BATCH
#define DI_LL_BATCH 8     // long rows (option long_lanes): column loads in flight per lane
#endif
#ifndef DI_LL_PIPE
#define DI_LL_PIPE 0      // 1: the next batch's loads issued before the current batch's REDs
#endif
#ifndef DI_ASYNC_MINB
#define DI_ASYNC_MINB 4
#endif
constexpr int kAsyncSmall = DI_ASYNC_SMALL;  // rows with <= this many links: a lane each
static_assert(kAsyncSmall < 256, "short-row length is packed in 8 bits");
constexpr int kAsyncMid = DI_ASYNC_MID;      // rows up to this: one 8-lane group each (list front)
constexpr int kAsyncChunk = DI_ASYNC_CHUNK;  // longer rows: chunks of this many links, one warp each

// Replicated accumulators for the hottest targets. Same-address fp64 REDs serialise in one L2
// slice; a node that receives a large share of all pushes (C3's Zipf targets: the top node gets
// 0.39 % of the links; C4's R-MAT top node 0.09 %) keeps its slice busy for a large part of the
// cycle and throttles every SM that has a RED queued behind it. On such a graph (top share >
// kReplShare) the upload places the kHotRanks hottest nodes at internal ids 0..kHotRanks-1
// (graph_build.cu, k_place); their REDs go to one of kCopies copies (chosen by warp), every copy
// in its own 128-B line (copies sharing a line serialise like one address: tools/micro/hot.cu,
// profiles/micro_hot.txt), and the last CTA of the cycle folds the copies into F.
constexpr int kRepl = kHotRanks;
constexpr int kCopies = kRepCopies;

// Hub items. On R-MAT graphs the hottest targets are also the largest rows (node 0 of C4 has
// ~240k out-links): pushed by the CTA that takes tile 0 they would make it the straggler of
// every cycle. Hot rows longer than kHubMin are therefore split into items of kHubItem links
// (built once by prepare_cycle): the CTA of tile 0 (claim 0) takes their fluid, publishes
// v = T d / o per hub row in hv[] and raises hub_flag; claims 1..n_hub are the items, pushed
// by whichever CTAs draw them once the flag is up; claims > n_hub are tiles 1, 2, ...
constexpr int64_t kHubMin = 8192;
constexpr int64_t kHubItem = 16384;

// Warm tier: a push to one of the warm ids is an fp64 add into the CTA's
// shared-memory accumulator (a CAS loop: sm_100a has no native shared fp64 add) instead of an L2
// RED; k_cycle flushes the accumulators into F when the CTA leaves the cycle. The warm ids are the
// hot ids [0, hot) (slots nw + j) and the ids hot + k * 2^shift, k < nw (slot k): the relabelling
// puts the warm ranks one every 2^shift ids (graph_build.cu k_place), so that every tile of the
// cycle keeps about the same work (warm rows are long: placed together they made one CTA the
// straggler of every cycle). On C4 the 4096 hottest ids take ~15 % of the link targets: that many
// fewer random requests reach the L2, whose request rate bounds the push
// (profiles/micro_redkind.txt).
template <bool ON>   // ON = false: the instantiations without a warm tier (no code for it)
struct WarmT {
  double *s;       // nw + hot accumulators (dynamic shared memory)
  int32_t hot;     // hot ids in the tier (0: off)
  uint32_t mask;   // 2^shift - 1
  uint32_t lim;    // nw << shift (0: off)
  int shift, nw;
};

template <bool ON>
__device__ __forceinline__ bool warm_take(const WarmT<ON> &w, int32_t j, double v) {
  if constexpr (!ON) return false;
  if (j < w.hot) {
    atomicAdd(w.s + w.nw + j, v);
    return true;
  }
  const uint32_t u = (uint32_t)(j - w.hot);
  if ((u & w.mask) == 0u && u < w.lim) {
    atomicAdd(w.s + (u >> w.shift), v);
    return true;
  }
  return false;
}

template <bool LOOPS, bool WON>
__device__ __forceinline__ void red_group_rep(double *__restrict__ F, double *__restrict__ rep,
                                              int hot_shift, int32_t hot_lim, int copy, int4 x,
                                              int64_t p0, int64_t beg, int64_t end, int32_t gi,
                                              double v, uint64_t fpol, const WarmT<WON> &w) {
  const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end && (!LOOPS || jj[c] != gi)) {
      const int32_t j = jj[c];
      if (warm_take(w, j, v))   // warm tier: the CTA's shared-memory accumulator
        ;
      else if (j < hot_lim)   // one of the hot ids 0..hot_lim-1 (0 when off)
        red_add_f64(rep + (int64_t)(copy * kRepl + j) * kRepStride, v);
      else
        red_add_f64_hint(F + j, v, fpol);
    }
  }
}

// DIST: targets are global internal ids; a target outside this rank's range gets a RED into the
// remote accumulator (push_remote, sweep.cuh).
template <bool LOOPS, bool DIST, bool WON>
__device__ __forceinline__ void push_group(const SweepArgs &a, const DistArgs &x, double *rep,
                                           int hot_shift, int32_t hot_lim, int copy, int4 q,
                                           int64_t p0, int64_t beg, int64_t end, int32_t gi,
                                           double v, uint64_t fpol, const WarmT<WON> &w) {
  if (!DIST) {
    red_group_rep<LOOPS>(a.F, rep, hot_shift, hot_lim, copy, q, p0, beg, end, gi, v, fpol, w);
    return;
  }
  const int32_t jj[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end && (!LOOPS || jj[c] != gi)) {
      const int64_t jl = (int64_t)jj[c] - a.lo;
      if (jl >= 0 && jl < a.n)
        red_add_f64_hint(a.F + jl, v, fpol);
      else
        push_remote(x, jj[c], v);
    }
  }
}

__device__ __forceinline__ double take_fluid(double *p) {
  return __longlong_as_double(
      (long long)atomicExch(reinterpret_cast<unsigned long long *>(p), 0ull));
}

__device__ __forceinline__ void st_cold(ColdRec *r, int32_t j, double v) {
  const long long b = __double_as_longlong(v);
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(r), "r"(j), "r"(0),
               "r"((int)(b & 0xffffffffll)), "r"((int)(b >> 32))
               : "memory");
}

// Cold bins. Every warp owns one chunk of kColdChunk records per bin at a time
// (shared memory: its start inside the bin's region, and the number of slots taken). A lane with
// a cold target takes a slot with one shared-memory atomic and stores its 16-B record; when a
// chunk runs out, the lanes that got no slot keep their records and the warp — at the end of the
// int4 group, where it is converged — records the full chunk's fill, reserves a fresh chunk for
// each exhausted bin (one global atomic per kColdChunk records) and retries them. Partially filled
// chunks record their fill at the end of the cycle; k_cold_apply reads the fills.
// Per-bin pointers (shared memory): the bin's region of records, its chunk fills, its counter.
// One GPU: the bins of target slices in the arena. Partitioned (compact remote path): bin p is
// owner p, the region this sender's cold records take in p's inbox (parity of the cycle).
__device__ __noinline__ void cold_refill(int nbins, int32_t *const *fptr,
                                         unsigned long long *const *tptr, int32_t *cnt,
                                         int32_t *base, int lane) {
  for (int b = lane; b < nbins; b += 32) {
    if (cnt[b] >= kColdChunk && tptr[b]) {   // (partitioned: no bin for the own range)
      if (base[b] >= 0) fptr[b][base[b] / kColdChunk] = kColdChunk;
      base[b] = (int32_t)atomicAdd(tptr[b], (unsigned long long)kColdChunk);
      cnt[b] = 0;
    }
  }
  __syncwarp();
}

__device__ __forceinline__ bool cold_put(ColdRec *const *cptr, int32_t *cnt, const int32_t *base,
                                         int b, int32_t j, double v) {
  const int p = atomicAdd(cnt + b, 1);
  if (p >= kColdChunk) return false;
  st_cold(cptr[b] + base[b] + p, j, v);
  return true;
}

// the records of an int4 group that found their chunk full (warp-collective; rare: once per
// kColdChunk records of a bin and warp); bins packed 6 bits per target. Scalar and shared-memory
// arguments only: a reference to the kernel's parameter block would make the compiler copy it
// to the stack.
__device__ __noinline__ void cold_retry(int nbins, ColdRec *const *cptr, int32_t *const *fptr,
                                        unsigned long long *const *tptr, int32_t *cnt,
                                        int32_t *base, int4 q, unsigned pending, unsigned bins,
                                        double v, int lane, int32_t dec, int32_t cw) {
  // the records' ids from the columns: q - dec on one GPU; partitioned, the owner-local id
  // q - dec - owner * cw (the column encoding, dist.cu k_encode_col)
  int32_t jj[4] = {q.x - dec, q.y - dec, q.z - dec, q.w - dec};
  for (int c = 0; c < 4; c++) jj[c] -= (int32_t)((bins >> (6 * c)) & 63u) * cw;
  while (__any_sync(0xffffffffu, pending != 0u)) {
    cold_refill(nbins, fptr, tptr, cnt, base, lane);
    for (int c = 0; c < 4; c++)
      if ((pending >> c) & 1u)
        if (cold_put(cptr, cnt, base, (int)((bins >> (6 * c)) & 63u), jj[c], v)) pending &= ~(1u << c);
  }
}

struct ColdSm {   // the warp's chunk state and the block's per-bin pointers (shared memory)
  int32_t *cnt, *base;
  ColdRec *const *cptr;
  int32_t *const *fptr;
  unsigned long long *const *tptr;
  // partitioned: a cold target's column is n + rsum + p * cw + (its id in owner p's range)
  // (dist.cu k_encode_col): the owner is one fp32 multiply (and at most one correction) away
  uint32_t cw;    // owner window (the largest range)
  float cinv;     // 1 / cw
  int64_t rsum;   // hot remote slots (sum of rt)
};

// COLD push of one int4 group (warp-collective: every lane calls it; `valid` = the lane has a
// group). One GPU: hot ids to the replicated accumulators, first-tier targets (j < cold_lo) a
// RED into F, cold targets a record of their slice's bin. Partitioned (DIST): local targets a RED
// into F, hot remote targets (the first rt[p] ids of owner p's range) a RED into the compact
// accumulator, colder remote targets a record into owner p's inbox.
template <bool LOOPS, bool DIST, bool WON>
__device__ __forceinline__ void push_group_cold(const SweepArgs &a, const DistArgs &x,
                                                double *__restrict__ rep, int32_t hot_lim, int copy,
                                                int4 q, int64_t p0, int64_t beg, int64_t end,
                                                bool valid, int32_t gi, double v, uint64_t fpol,
                                                const ColdSm &cs, int lane, const WarmT<WON> &w) {
  unsigned pending = 0u, bins = 0u;
  auto one = [&](int c, int32_t j) {
    const int64_t p = p0 + c;
    if (!(valid && p >= beg && p < end && (!LOOPS || j != gi))) return;
    if (DIST) {
      // the compact path's encoded column (dist.cu k_encode_col): [0, n) local ids, then the hot
      // remote targets' accumulator slots, then n + R + global id for colder remote targets
      const uint32_t e = (uint32_t)j;
      if (e < (uint32_t)a.n) {
        red_add_f64_hint(a.F + e, v, fpol);
      } else if (e < (uint32_t)(a.n + cs.rsum)) {
        red_add_f64_hint(x.racc + (e - (uint32_t)a.n), v, fpol);
      } else {
        const uint32_t u = e - (uint32_t)(a.n + cs.rsum);
        int pp = (int)((float)u * cs.cinv);   // the owner, within one of the quotient
        int32_t lj = (int32_t)(u - (uint32_t)pp * cs.cw);
        if (lj < 0) {
          pp--;
          lj += (int32_t)cs.cw;
        } else if (lj >= (int32_t)cs.cw) {
          pp++;
          lj -= (int32_t)cs.cw;
        }
        if (!cold_put(cs.cptr, cs.cnt, cs.base, pp, lj, v)) {
          pending |= 1u << c;
          bins |= (unsigned)pp << (6 * c);
        }
      }
    } else if ((int64_t)j >= a.cold_lo) {
      const int bb = (int)(((int64_t)j - a.cold_lo) >> a.cold_shift);
      if (!cold_put(cs.cptr, cs.cnt, cs.base, bb, j, v)) {
        pending |= 1u << c;
        bins |= (unsigned)bb << (6 * c);
      }
    } else if (warm_take(w, j, v)) {
    } else if (j < hot_lim) {
      red_add_f64(rep + (int64_t)(copy * kRepl + j) * kRepStride, v);
    } else {
      red_add_f64_hint(a.F + j, v, fpol);
    }
  };
  // not unrolled: the COLD kernel's code must stay small enough for the instruction cache (with
  // the four targets unrolled at every call site, half the stall samples of the single-GPU kernel
  // were no_instruction; unrolled, the partitioned kernel took 1801 instead of 1118 us per cycle)
#pragma unroll 1
  for (int c = 0; c < 4; c++) one(c, c == 0 ? q.x : (c == 1 ? q.y : (c == 2 ? q.z : q.w)));
  if (__any_sync(0xffffffffu, pending != 0u))
    cold_retry(DIST ? x.bd.world : a.cold_nbins, cs.cptr, cs.fptr, cs.tptr, cs.cnt, cs.base, q,
               pending, bins, v, lane, DIST ? (int32_t)(a.n + cs.rsum) : 0, DIST ? (int32_t)cs.cw : 0);
}

// TEST (di_test_cycle, include/di_test.h): the selection records (T, v) per node in a.rec_T /
// a.rec_v instead of pushing, so that the select-and-take step of this kernel can be compared bit
// for bit with the oracle's bulk sweep on a frozen F (no push: nothing changes F during the cycle)
// COLD: cold bins on (single GPU, F several times the L2)
template <bool LOOPS, bool DIST, bool TEST = false, bool COLD = false, bool WARM = false>
__global__ void __launch_bounds__(kAsyncThreads, DI_ASYNC_MINB) k_cycle(const SweepArgs a, const DistArgs x) {
  constexpr int NW = kAsyncThreads / 32;
  constexpr int NCB = COLD ? kColdBins : 1;
  __shared__ int32_t s_ccb[NW][NCB], s_cce[NW][NCB];   // COLD: per-warp chunk (slots taken, start)
  __shared__ ColdRec *s_cptr[NCB];
  __shared__ int32_t *s_fptr[NCB];
  __shared__ unsigned long long *s_tptr[NCB];
  __shared__ int64_t s_rb[kCycTile];   // long rows of the tile: first link
  __shared__ int32_t s_ro[kCycTile];   // #links
  __shared__ double s_rv[kCycTile];    // v = T d / o
  __shared__ int32_t s_ri[kCycTile];   // local node id
  __shared__ int32_t s_rp[kCycTile + 1];  // exclusive chunk prefix
  __shared__ int16_t s_si[kCycTile];   // short rows of the tile: local node id
  __shared__ double s_sv[kCycTile];    //   and v
  __shared__ int64_t s_sb[kCycTile];   //   and first link << 8 | #links
  __shared__ int s_nrows, s_nmid, s_nsmall, s_nchunks, s_claim, s_mclaim, s_sclaim;
  __shared__ int64_t s_tile;
  __shared__ int s_item;
  __shared__ bool s_last;
  __shared__ double s_red[NW][4];
  __shared__ long long s_ired[NW][3];
  extern __shared__ double s_warm[];   // warm tier accumulators (dynamic shared memory)

  Scalars *sc = a.sc;
  if (sc->stop) return;
  unsigned long long t_begin = 0;
  if (a.times && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hot_shift = a.hot_shift;
  const int32_t hot_lim = hot_shift >= 0 ? hot_shift : 0;   // a.hot_shift = hot-id count here
  const int copy = (blockIdx.x * (kAsyncThreads / 32) + warp) % kCopies;
  double *rep = a.rep;
  double *hv = rep + kCopies * kRepl * kRepStride;  // hub rows' v (valid when a.n_hub > 0)
  const unsigned hub_tag = sc->hub_want + 1u;       // hub_flag value of this cycle
  const double r = sc->r, d = sc->d;
  const bool cyc = (sc->variant == DI_CYC) || sc->guard;
  double t = (a.L_total > 0.0) ? r / a.L_total : 0.0;  // r/L once per cycle (G3, G4)
  if (sc->alpha != 1.0) t = __dmul_rn(t, sc->alpha);  // F4 threshold scale (1 = the paper's rule)
  const uint64_t pol = policy_evict_first();
  const uint64_t fpol = a.red_hint ? policy_evict_last() : policy_evict_normal();
  const int32_t *__restrict__ col = a.col;
  double *__restrict__ F = a.F;
  double acc_tk = 0.0, acc_s = 0.0, acc_e = 0.0;
  long long acc_sel = 0, acc_nd = 0, acc_lk = 0;
  int32_t *ccb = s_ccb[warp], *cce = s_cce[warp];
  const int cnb = DIST ? x.bd.world : a.cold_nbins;
  if (COLD) {
    for (int b = lane; b < NCB; b += 32) {
      ccb[b] = kColdChunk;   // slots taken in the current chunk (full: none yet)
      cce[b] = -1;           // its start inside the bin's region (-1: none)
    }
    const int b = threadIdx.x;
    if (b < NCB) {
      s_cptr[b] = nullptr;
      s_fptr[b] = nullptr;
      s_tptr[b] = nullptr;
      if (!DIST && b < a.cold_nbins) {
        s_cptr[b] = a.cold_rec + a.cold_off[b];
        s_fptr[b] = a.cold_fill + a.cold_off[b] / kColdChunk;
        s_tptr[b] = a.cold_top + 16 * b;
      } else if (DIST && b < x.bd.world && b != x.rank) {
        const int64_t slot = 2 * (int64_t)x.rank + x.ipar;
        s_cptr[b] = reinterpret_cast<ColdRec *>(x.inbox[b] + x.cold_off0) + slot * x.ccap;
        s_fptr[b] = reinterpret_cast<int32_t *>(x.inbox[b] + x.fill_off0) + slot * (x.ccap / kColdChunk);
        s_tptr[b] = x.ctop + 16 * b;
      }
    }
  }
  const int nwarm = (WARM && !DIST) ? a.warm : 0;   // slots: nwarm warm-rank ids, then the hot ids
  const WarmT<WARM> wt{s_warm, nwarm > 0 ? a.warm_hot : 0, (1u << a.warm_shift) - 1u,
                 nwarm > 0 ? (uint32_t)nwarm << a.warm_shift : 0u, a.warm_shift, nwarm};
  const int nslots = (WARM && nwarm > 0) ? nwarm + a.warm_hot : 0;
  int tiles_done = 0;
  for (int k = threadIdx.x; k < nslots; k += kAsyncThreads) s_warm[k] = 0.0;   // (the loop's
                                                                               //  first barrier)
  const ColdSm cs{ccb, cce, s_cptr, s_fptr, s_tptr, (COLD && DIST) ? (uint32_t)x.cwin : 1u,
                  (COLD && DIST) ? 1.0f / (float)x.cwin : 1.0f, (COLD && DIST) ? x.hoff[x.bd.world] : 0};
  // the row's own id in the column's numbering (self-loop test): the compact path's columns are
  // encoded with local ids, the others hold global ids
  const int64_t gbase = (COLD && DIST) ? 0 : a.lo;

  for (;;) {
    if (threadIdx.x == 0) {
      // (option dist_parts: this launch takes the claims [claim_lo, claim_hi) of the rank's cycle)
      const int64_t c = (int64_t)atomicAdd(&sc->tile_next, 1u) + a.claim_lo;
      int64_t tl = c;
      int it = -1;
      if (c > 0 && a.n_hub > 0) {  // claims 1..n_hub: hub items; then tiles 1, 2, ...
        if (c <= a.n_hub) {
          it = (int)(c - 1);
          tl = 0;
        } else {
          tl = c - a.n_hub;
        }
      }
      if (a.claim_hi >= 0 && c >= a.claim_hi) {   // past this launch's window
        tl = a.ntiles;
        it = -1;
      }
      if (COLD && it < 0 && tl < a.ntiles) {
        // the first-tier (hot) tiles are spread evenly over the cycle instead of all coming
        // first: a hot node is then visited after the pushes of the tiles before it, as in the
        // one-tier striped order (claim 0 stays tile 0: the hub rows' tile). Bijection of
        // [0, ntiles): claim c is hot iff ceil((c+1)H/T) > ceil(cH/T)
        const int64_t H = a.cold_hot_tiles, T = a.ntiles;
        const int64_t h0 = (tl * H + T - 1) / T, h1 = ((tl + 1) * H + T - 1) / T;
        tl = (h1 > h0) ? h0 : H + (tl - h0);
      }
      s_tile = tl;
      s_item = it;
      s_nrows = 0;
      s_nmid = 0;
      s_nsmall = 0;
      s_claim = 0;
      s_mclaim = 0;
      s_sclaim = 0;
    }
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    if (s_item >= 0) {  // ---- a hub item: links [beg, end) of hot row `row`, v from tile 0
      if (threadIdx.x == 0) {
        const int64_t *h = a.hub + 3 * (int64_t)s_item;
        const int64_t row = h[0], beg = h[1], end = h[2];
        while (ld_acquire_u32(&sc->hub_flag) != hub_tag) __nanosleep(64);
        const double v = __ldcg(hv + row);
        if (v != 0.0) {
          s_rb[kCycTile - 1] = beg;
          s_ro[kCycTile - 1] = (int32_t)(end - beg);
          s_rv[kCycTile - 1] = v;
          s_ri[kCycTile - 1] = (int32_t)row;
          s_nrows = 1;
        }
      }
    } else {
    // ---- select: kCycItems consecutive nodes per thread, F and row extents
    const int64_t base = tile * (int64_t)kCycTile + (int64_t)threadIdx.x * kCycItems;
    double f[kCycItems];
    int64_t rb[kCycItems + 1];
    int kl[kCycItems];
    if (kCycItems % 2 == 0 && base + kCycItems <= a.n) {  // vectorised: 2 x double2 (F, L2 only: REDs land there) and
                                    // 2 x longlong2 (row extents) + the next row's start
#pragma unroll
      for (int h = 0; h < kCycItems / 2; h++) {
        const double2 fp = __ldcg(reinterpret_cast<const double2 *>(F + base) + h);
        const longlong2 rp = ld_i64x2_stream(a.row_ptr + base + 2 * h, pol);
        f[2 * h] = fp.x;
        f[2 * h + 1] = fp.y;
        rb[2 * h] = rp.x;
        rb[2 * h + 1] = rp.y;
      }
      rb[kCycItems] = ld_i64_stream(a.row_ptr + base + kCycItems, pol);
#pragma unroll
      for (int j = 0; j < kCycItems; j++) kl[j] = LOOPS ? a.kloop[base + j] : 0;
    } else {
#pragma unroll
      for (int j = 0; j < kCycItems; j++) {
        const int64_t i = base + j;
        f[j] = (i < a.n) ? __ldcg(F + i) : 0.0;
        rb[j] = (i < a.n) ? a.row_ptr[i] : 0;
        kl[j] = (LOOPS && i < a.n) ? a.kloop[i] : 0;
      }
      rb[kCycItems] = base < a.n ? a.row_ptr[min(base + kCycItems, a.n)] : 0;
    }
    // the selection test for the thread's nodes first, then all their exchanges in flight together
    // (one round trip per tile instead of one per selected node)
    int o4[kCycItems];
    bool hub4[kCycItems];
    double T04[kCycItems];
#pragma unroll
    for (int j = 0; j < kCycItems; j++) {
      const int64_t i = base + j;
      o4[j] = -1;  // not selected
      hub4[j] = false;
      if (i >= a.n) continue;
      const int64_t rend = (i + 1 < a.n) ? (j + 1 < kCycItems ? rb[j + 1] : rb[kCycItems])
                                         : a.row_ptr[a.n];
      const int o = (int)(rend - rb[j]);
      hub4[j] = i < hot_lim && o > kHubMin && a.n_hub > 0;      // pushed as hub items
      const double thr = cyc ? 0.0 : __dmul_rn(t, (double)o);  // (r/L)*out[i]
      if (f[j] > thr) o4[j] = o;                                // strict '>'
    }
#pragma unroll
    for (int j = 0; j < kCycItems; j++) {
#if DI_TAKE_SUB
      // take exactly the fluid the test saw: F_i -= f (a RED, nothing to wait for); fluid that
      // arrived since the read stays in F_i for the next visit
      T04[j] = 0.0;
      if (o4[j] >= 0 && !TEST) {
        T04[j] = f[j];
        red_add_f64(F + base + j, -f[j]);
      } else if (o4[j] >= 0) {
        T04[j] = take_fluid(F + base + j);
      }
#else
      T04[j] = (o4[j] >= 0) ? take_fluid(F + base + j) : 0.0;  // >= f[j]: only REDs add meanwhile
#endif
    }
#pragma unroll
    for (int j = 0; j < kCycItems; j++) {
      if (o4[j] < 0) {
        if (hub4[j]) {  // not selected: its items push nothing this cycle
          hv[base + j] = 0.0;
          __threadfence();
        }
        continue;
      }
      const int64_t i = base + j;
      const int o = o4[j];
      const double T0 = T04[j];
      double T = T0;
      if (LOOPS && kl[j] > 0) {                                 // P:259-263 with k copies (G6)
        const double od = (double)o;
        T = __ddiv_rn(__dmul_rn(T0, od), __dsub_rn(od, __dmul_rn((double)kl[j], d)));
      }
      red_add_f64_hint(a.H + i, T, pol);                        // P:264 (streamed: evict_first)
      acc_tk += T0;
      acc_sel++;
      if (o == 0) {
        acc_e += T;
        if (TEST) {
          a.rec_T[i] = T;
          a.rec_v[i] = 0.0;
        }
        continue;
      }
      const double v = __ddiv_rn(__dmul_rn(T, d), (double)o);
      acc_s += __dmul_rn(v, (double)(o - kl[j]));
      acc_lk += o;
      acc_nd++;
      if (TEST) {
        a.rec_T[i] = T;
        a.rec_v[i] = v;
        continue;
      }
      if (hub4[j]) {
        hv[i] = v;
        __threadfence();
      } else if (o <= kAsyncSmall) {   // short rows: their own list, a lane each (balanced below)
        const int p = atomicAdd(&s_nsmall, 1);
        s_si[p] = (int16_t)(base + j - tile * kCycTile);
        s_sv[p] = v;
        s_sb[p] = (rb[j] << 8) | (int64_t)o;
      } else {  // mid rows at the front of the list, long rows at its back
        const int p = (o <= kAsyncMid) ? atomicAdd(&s_nmid, 1) : kCycTile - 1 - atomicAdd(&s_nrows, 1);
        s_rb[p] = rb[j];
        s_ro[p] = o;
        s_rv[p] = v;
        s_ri[p] = (int32_t)(base + j - tile * kCycTile);
      }
    }
    }
    __syncthreads();
    if (tile == 0 && s_item < 0 && a.n_hub > 0 && threadIdx.x == 0) {  // hv[] complete: release
      __threadfence();
      st_release_u32(&sc->hub_flag, hub_tag);
    }
    // ---- long rows (list back: row k at kCycTile-1-k): chunk prefix (warp 0), then the CTA's
    //      warps claim chunks; then mid rows (list front), four per warp step
    const int nrows = s_nrows;
    if (nrows > 0) {
      if (warp == 0) {
        const int per = (nrows + 31) / 32;
        const int r0 = lane * per, r1 = min(nrows, r0 + per);
        int sum = 0;
        for (int k = r0; k < r1; k++) sum += (s_ro[kCycTile - 1 - k] + kAsyncChunk - 1) / kAsyncChunk;
        int incl = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        int run = incl - sum;
        for (int k = r0; k < r1; k++) {
          s_rp[k] = run;
          run += (s_ro[kCycTile - 1 - k] + kAsyncChunk - 1) / kAsyncChunk;
        }
        if (lane == 31) {
          s_nchunks = incl;
          s_rp[nrows] = incl;
        }
      }
      __syncthreads();
      const int nch = s_nchunks;
      for (;;) {
        int c = 0;
        if (lane == 0) c = atomicAdd(&s_claim, 1);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= nch) break;
        int lo = 0, hi = nrows - 1;  // last row with s_rp[row] <= c
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_rp[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int slot = kCycTile - 1 - lo;
        const int64_t rbeg = s_rb[slot];
        const int64_t beg = rbeg + (int64_t)(c - s_rp[lo]) * kAsyncChunk;
        const int64_t end = min(rbeg + (int64_t)s_ro[slot], beg + kAsyncChunk);
        const double v = s_rv[slot];
        const int32_t gi = LOOPS ? (int32_t)(tile * kCycTile + s_ri[slot] + gbase) : -1;
        const int64_t a0 = beg & ~3ll;
        const int nvec = (int)((end - a0 + 3) >> 2);
        if (!COLD && !DIST && a.long_lanes) {
          // lane-consecutive targets: lane l takes links beg + 32u + l, so the 32 REDs of one
          // instruction go to 32 consecutive (sorted) targets of the row, which share L2 lines
          // where the row is dense in the hot ids; scalar coalesced loads, no masked lanes
          constexpr int NB = DI_LL_BATCH;   // loads in flight per lane
#if DI_LL_PIPE
          // software-pipelined: the next batch's column loads are issued before this batch's REDs
          int32_t nx[NB];
#pragma unroll
          for (int u = 0; u < NB; u++) {
            const int64_t p = beg + 32 * u + lane;
            nx[u] = p < end ? ld_col(col + p, pol) : -1;
          }
#endif
          for (int64_t p0 = beg; p0 < end; p0 += 32 * NB) {
            int32_t jj[NB];
#if DI_LL_PIPE
#pragma unroll
            for (int u = 0; u < NB; u++) {
              jj[u] = nx[u];
              const int64_t p = p0 + 32 * (NB + u) + lane;
              nx[u] = p < end ? ld_col(col + p, pol) : -1;
            }
#else
#pragma unroll
            for (int u = 0; u < NB; u++) {
              const int64_t p = p0 + 32 * u + lane;
              jj[u] = p < end ? ld_col(col + p, pol) : -1;
            }
#endif
#pragma unroll
            for (int u = 0; u < NB; u++) {
              const int32_t j = jj[u];
              if (j >= 0 && (!LOOPS || j != gi)) {
                if (warm_take(wt, j, v))
                  ;
                else if (j < hot_lim)
                  red_add_f64(rep + (int64_t)(copy * kRepl + j) * kRepStride, v);
                else
                  red_add_f64_hint(F + j, v, fpol);
              }
            }
          }
          continue;
        }
        for (int vb = 0; vb < nvec; vb += 128) {
          int4 xq[4];
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const int vi = vb + 32 * k + lane;
            xq[k] = make_int4(0, 0, 0, 0);
            if (vi < nvec) xq[k] = ld_col4(col + a0 + 4 * (int64_t)vi, pol);
          }
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const int vi = vb + 32 * k + lane;
            if constexpr (COLD)
              push_group_cold<LOOPS, DIST>(a, x, rep, hot_lim, copy, xq[k], a0 + 4 * (int64_t)vi, beg, end,
                                     vi < nvec, gi, v, fpol, cs, lane, wt);
            else if (vi < nvec)
              push_group<LOOPS, DIST>(a, x, rep, hot_shift, hot_lim, copy, xq[k], a0 + 4 * (int64_t)vi,
                                      beg, end, gi, v, fpol, wt);
          }
        }
      }
    }
    // short rows (<= kAsyncSmall links, <= 5 int4 groups): 32 per warp claim, one per lane
    const int nsmall = s_nsmall;
    if (nsmall > 0) {
      const int64_t tb = tile * (int64_t)kCycTile;
      for (;;) {
        int q = 0;
        if (lane == 0) q = atomicAdd(&s_sclaim, 32);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= nsmall) break;
        const int k = q + lane;
        if constexpr (COLD) {   // warp-collective pushes: every lane runs the NG groups
          const bool has = k < nsmall;
          const int li = has ? s_si[k] : 0;
          const double v = has ? s_sv[k] : 0.0;
          const int64_t sb = has ? s_sb[k] : 0;
          const int64_t beg = sb >> 8, end = beg + (sb & 255), a0 = beg & ~3ll;
          const int nvec = has ? (int)((end - a0 + 3) >> 2) : 0;
          const int32_t gi = LOOPS ? (int32_t)(tb + li + gbase) : -1;
          // only as many groups as the warp's longest short row needs (warp-uniform), not the
          // kAsyncSmall bound: most short rows have 1-2 int4 groups
          const int umax = __reduce_max_sync(0xffffffffu, nvec);
#pragma unroll 1
          for (int u = 0; u < umax; u++) {
            const int4 xg = u < nvec ? ld_col4(col + a0 + 4 * u, pol) : make_int4(0, 0, 0, 0);
            push_group_cold<LOOPS, DIST>(a, x, rep, hot_lim, copy, xg, a0 + 4 * u, beg, end, u < nvec, gi,
                                         v, fpol, cs, lane, wt);
          }
        } else if (k < nsmall) {
          const int li = s_si[k];
          const double v = s_sv[k];
          const int64_t sb = s_sb[k];
          const int64_t beg = sb >> 8, end = beg + (sb & 255), a0 = beg & ~3ll;
          const int nvec = (int)((end - a0 + 3) >> 2);
          const int32_t gi = LOOPS ? (int32_t)(tb + li + gbase) : -1;
          constexpr int NG = (kAsyncSmall + 6) / 4;   // aligned int4 groups of a short row
          int4 xs[NG];
#pragma unroll
          for (int u = 0; u < NG; u++) {
            xs[u] = make_int4(0, 0, 0, 0);
            if (u < nvec) xs[u] = ld_col4(col + a0 + 4 * u, pol);
          }
#pragma unroll
          for (int u = 0; u < NG; u++)
            if (u < nvec)
              push_group<LOOPS, DIST>(a, x, rep, hot_shift, hot_lim, copy, xs[u], a0 + 4 * u, beg,
                                      end, gi, v, fpol, wt);
        }
      }
    }
    const int nmid = s_nmid;
    if (nmid > 0) {
      const int sub = lane & 7;
      for (;;) {
        int q = 0;
        if (lane == 0) q = atomicAdd(&s_mclaim, 4);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= nmid) break;
        const int k = q + (lane >> 3);
        if constexpr (COLD) {   // warp-collective: every lane runs the warp's longest row's steps
          const bool has = k < nmid;
          const int64_t beg = has ? s_rb[k] : 0, end = has ? beg + s_ro[k] : 0, a0 = beg & ~3ll;
          const int nvec = has ? (int)((end - a0 + 3) >> 2) : 0;
          const double v = has ? s_rv[k] : 0.0;
          const int32_t gi = LOOPS && has ? (int32_t)(tile * kCycTile + s_ri[k] + gbase) : -1;
          const int maxn = __reduce_max_sync(0xffffffffu, nvec);
          for (int b0 = 0; b0 < maxn; b0 += 16) {
            const int vb = b0 + sub;
            int4 x0 = make_int4(0, 0, 0, 0), x1 = make_int4(0, 0, 0, 0);
            if (vb < nvec) x0 = ld_col4(col + a0 + 4 * (int64_t)vb, pol);
            if (vb + 8 < nvec) x1 = ld_col4(col + a0 + 4 * (int64_t)(vb + 8), pol);
            push_group_cold<LOOPS, DIST>(a, x, rep, hot_lim, copy, x0, a0 + 4 * (int64_t)vb, beg, end, vb < nvec,
                                   gi, v, fpol, cs, lane, wt);
            push_group_cold<LOOPS, DIST>(a, x, rep, hot_lim, copy, x1, a0 + 4 * (int64_t)(vb + 8), beg, end,
                                   vb + 8 < nvec, gi, v, fpol, cs, lane, wt);
          }
        } else if (k < nmid) {
          const int64_t beg = s_rb[k], end = beg + s_ro[k], a0 = beg & ~3ll;
          const int nvec = (int)((end - a0 + 3) >> 2);   // <= 33
          const double v = s_rv[k];
          const int32_t gi = LOOPS ? (int32_t)(tile * kCycTile + s_ri[k] + gbase) : -1;
          for (int vb = sub; vb < nvec; vb += 16) {
            const int4 x0 = ld_col4(col + a0 + 4 * (int64_t)vb, pol);
            int4 x1 = make_int4(0, 0, 0, 0);
            if (vb + 8 < nvec) x1 = ld_col4(col + a0 + 4 * (int64_t)(vb + 8), pol);
            push_group<LOOPS, DIST>(a, x, rep, hot_shift, hot_lim, copy, x0, a0 + 4 * (int64_t)vb, beg, end,
                                 gi, v, fpol, wt);
            if (vb + 8 < nvec)
              push_group<LOOPS, DIST>(a, x, rep, hot_shift, hot_lim, copy, x1, a0 + 4 * (int64_t)(vb + 8),
                                   beg, end, gi, v, fpol, wt);
          }
        }
      }
    }
    __syncthreads();
    // option warm_flush = k: the warm accumulators go to F every k tiles of this CTA too (the
    // barrier above: no push in flight; the next claim's barrier orders the zeroing)
    if (nslots > 0 && a.warm_flush > 0 && ++tiles_done % a.warm_flush == 0)
      for (int k = threadIdx.x; k < nslots; k += kAsyncThreads) {
        const double w = s_warm[k];
        if (w != 0.0) {
          s_warm[k] = 0.0;
          red_add_f64_hint(F + (k < nwarm ? (int64_t)wt.hot + ((int64_t)k << wt.shift) : (int64_t)(k - nwarm)),
                           w, fpol);
        }
      }
  }
  // the warm accumulators into F (every push of this CTA is done: the loop ends at a barrier);
  // before the ticket, so that the cycle's last CTA sees all of the cycle's fluid in F
  for (int k = threadIdx.x; k < nslots; k += kAsyncThreads) {
    const double w = s_warm[k];
    const int64_t j = k < nwarm ? (int64_t)wt.hot + ((int64_t)k << wt.shift) : (int64_t)(k - nwarm);
    if (w != 0.0) red_add_f64_hint(F + j, w, fpol);
  }
  if (COLD && lane == 0) {  // the warp's open chunks: their fill for the apply kernels
    for (int b = 0; b < cnb; b++)
      if (cce[b] >= 0) s_fptr[b][cce[b] / kColdChunk] = min(ccb[b], kColdChunk);
  }
  // ---- this CTA's sums (fixed order inside the CTA) -> ppartials[blockIdx.x]
  acc_tk = warp_sum(acc_tk);
  acc_s = warp_sum(acc_s);
  acc_e = warp_sum(acc_e);
  acc_sel = warp_sum(acc_sel);
  acc_nd = warp_sum(acc_nd);
  acc_lk = warp_sum(acc_lk);
  if (lane == 0) {
    s_red[warp][0] = acc_tk;
    s_red[warp][1] = acc_s;
    s_red[warp][2] = acc_e;
    s_ired[warp][0] = acc_sel;
    s_ired[warp][1] = acc_nd;
    s_ired[warp][2] = acc_lk;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x[3] = {0.0, 0.0, 0.0};
    long long c[3] = {0, 0, 0};
    for (int w = 0; w < NW; w++) {
      for (int k = 0; k < 3; k++) x[k] += s_red[w][k];
      for (int k = 0; k < 3; k++) c[k] += s_ired[w][k];
    }
    // slot layout of slice_partials: q, s, e, taken, sel, nd, links, 0 (q unused here)
    double *o = a.ppartials + 8 * (int64_t)blockIdx.x;
    reinterpret_cast<double2 *>(o)[0] = make_double2(0.0, x[1]);
    reinterpret_cast<double2 *>(o)[1] = make_double2(x[2], x[0]);
    reinterpret_cast<longlong2 *>(o)[2] = make_longlong2(c[0], c[1]);
    reinterpret_cast<longlong2 *>(o)[3] = make_longlong2(c[2], 0);
    if (a.times) {
      unsigned long long t_end;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      unsigned long long *tp = a.times + 2 * ((int64_t)(sc->sweeps & 63) * gridDim.x + blockIdx.x);
      tp[0] = t_begin;
      tp[1] = t_end;
    }
    __threadfence();
    s_last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (hot_shift >= 0) {  // fold the replicated accumulators into F, clear them
    for (int k = threadIdx.x; k < hot_lim; k += kAsyncThreads) {
      double acc = 0.0;
      for (int c = 0; c < kCopies; c++) {
        double *p = rep + (int64_t)(c * kRepl + k) * kRepStride;
        acc += __ldcg(p);
        *p = 0.0;
      }
      if (acc != 0.0) F[k] += acc;
    }
  }
  const SweepSums sm = reduce_partials(a, gridDim.x, kAsyncThreads);
  if (DIST) {  // this rank's sums; k_compact_remote counts, the host exchanges, finalize applies
    if (threadIdx.x == 0) {
      x.dsum[0] = 0.0;
      x.dsum[1] = sm.s;
      x.dsum[2] = sm.e;
      x.dsum[3] = sm.taken;
      x.isum[0] = sm.sel;
      x.isum[1] = sm.nd;
      x.isum[2] = sm.lk;
      x.isum[3] = a.n;
      sc->tile_next = 0;
      sc->ticket = 0;
      sc->hub_want = hub_tag;
    }
    return;
  }
  if (threadIdx.x != 0) return;
  // ---- the cycle's effect (P:278-283 stop test, G5 guard)
  volatile Scalars *vs = a.sc;
  const int variant = vs->variant;
  const double r_next = __dadd_rn(__dsub_rn(r, sm.taken), sm.s);
  const double e_tot = vs->e + sm.e;
  const int64_t sw = vs->sweeps;
  if (vs->trace && sw < kLogCap) {
    a.log_r[sw] = r;
    a.log_sel[sw] = sm.sel;
    a.log_links[sw] = sm.lk;
    a.log_mode[sw] = 0;
  }
  if (vs->guard && variant != DI_CYC) vs->guards = vs->guards + 1;
  vs->e = e_tot;
  vs->e_sw = sm.e;
  vs->s = sm.s;
  vs->q = __dsub_rn(r, sm.taken);
  vs->r = r_next;
  vs->sweeps = sw + 1;
  vs->selected_total = vs->selected_total + sm.sel;
  vs->selected_nd_total = vs->selected_nd_total + sm.nd;
  vs->links_total = vs->links_total + sm.lk;
  vs->scanned_total = vs->scanned_total + a.n;
  const double err = vs->paper_err ? r_next / (1.0 - d - d * e_tot) : r_next;
  const int stop = err <= vs->tol;
  vs->stop = stop;
  vs->guard = (sm.sel == 0 && !stop && variant == DI_SOP) ? 1 : 0;
  vs->tile_next = 0;
  vs->hub_want = hub_tag;
  vs->ticket = 0;
}

// Cold bins, after the cycle: the records of bin 0, then bin 1, ... (every block takes a contiguous
// share of each bin, so the grid walks the bins together and the slice of F being updated stays
// in L2), each a RED into F; the last block rewinds the bins. Chunks past their fill are skipped.
// The grid is co-resident (at most the resident blocks of the device) and the blocks meet at a
// barrier between two bins, so that the whole grid works on one slice of F at a time.
#ifndef DI_APPLY_UNROLL
#define DI_APPLY_UNROLL 4
#endif
constexpr int kApplyUnroll = DI_APPLY_UNROLL;

__global__ void __launch_bounds__(256) k_cold_apply(double *__restrict__ F, const ColdRec *__restrict__ rec,
                                                    const int64_t *__restrict__ off,
                                                    unsigned long long *top,
                                                    const int32_t *__restrict__ fill, int nbins) {
  __shared__ bool s_last;
  const uint64_t pol = policy_evict_first();
  unsigned int *bar = reinterpret_cast<unsigned int *>(top + 16 * kColdBins) + 32;
  for (int b = 0; b < nbins; b++) {
    if (b > 0) {  // grid barrier: every block done with bin b - 1
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned want = (unsigned)b * gridDim.x;
        while (ld_acquire_u32(bar) < want) __nanosleep(32);
      }
      __syncthreads();
    }
    const int64_t m = (int64_t)*reinterpret_cast<volatile unsigned long long *>(top + 16 * b);
    if (m == 0) continue;
    const int64_t base = off[b];
    const int64_t per = (m + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = r0 + per < m ? r0 + per : m;
    // kApplyUnroll records per thread in flight (loads first, then the REDs): the apply is
    // latency-bound on the record loads (ncu C5: 10 % issue active, long_scoreboard stalls)
    constexpr int U = kApplyUnroll;
    for (int64_t rb = r0 + threadIdx.x; rb < r1; rb += (int64_t)U * blockDim.x) {
      int4 q[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t r = rb + (int64_t)u * blockDim.x;
        const int64_t gr = base + r;   // regions are chunk-aligned
        ok[u] = r < r1 && (int)(r % kColdChunk) < __ldg(fill + gr / kColdChunk);
        q[u] = make_int4(0, 0, 0, 0);
        if (ok[u])
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                       : "=r"(q[u].x), "=r"(q[u].y), "=r"(q[u].z), "=r"(q[u].w)
                       : "l"(rec + gr), "l"(pol));
      }
#pragma unroll
      for (int u = 0; u < U; u++)
        if (ok[u]) red_add_f64(F + q[u].x, __hiloint2double(q[u].w, q[u].z));
    }
  }
  __syncthreads();
  unsigned int *ticket = reinterpret_cast<unsigned int *>(top + 16 * kColdBins);
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x < nbins) top[16 * threadIdx.x] = 0ull;
  if (threadIdx.x == 0) {
    *ticket = 0u;
    *bar = 0u;   // every block has passed its last barrier (they all reached the ticket)
  }
}

// cold-target counts per bin (static: the CSR), for the bin regions of the arena
__global__ void k_cold_hist(const int32_t *__restrict__ col, int64_t L, int64_t cold_lo, int shift,
                            unsigned long long *cnt) {
  __shared__ unsigned int h[kColdBins];
  if (threadIdx.x < kColdBins) h[threadIdx.x] = 0u;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[k];
    if (j >= cold_lo) atomicAdd(&h[(j - cold_lo) >> shift], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kColdBins && h[threadIdx.x]) atomicAdd(cnt + threadIdx.x, (unsigned long long)h[threadIdx.x]);
}

}  // namespace

// number of hot ids (replicated accumulators) for this graph, or -1 when off
static int hot_shift_of(const Graph &g) {
  return (g.reordered && g.hot_acc && !g.partitioned && g.hot_count > 0) ? (int)g.hot_count : -1;
}

static int cycle_grid(const Graph &g);
static void warm_init();

// cold bins: the arena of bin regions (cold in-links of the slice + one chunk per warp of the
// grid), chunk fills and counters; once per graph (the CSR is static)
static di_status prepare_cold(Graph &g) {
  if (g.cold_rec || g.partitioned || !(g.cold_lo < g.n)) return DI_OK;
  const int64_t ncold = g.n - g.cold_lo;
  // auto: slices of about the L2's size in F (C5: 2^24 nodes = 134 MB, 8 bins). Fewer, larger bins
  // won over L2-resident slices: every warp keeps one open chunk per bin, whose partly written
  // lines sit in the L2 beside the first tier (31 bins x 4736 warps ~ 19 MB of them); C5 623.7 /
  // 592.6 / 584.3 / 629.3 / 755.0 / 979.7 ms with 2^22 ... 2^27-node slices
  // (profiles/r2/c5_cold_shift.txt). The option cold_shift forces the slice size.
  int s = g.cold_shift_opt > 0 ? g.cold_shift_opt : kColdMinShift;
  if (g.cold_shift_opt <= 0)
    while ((8ll << s) < g.l2_bytes) s++;
  while ((((ncold + (1ll << s) - 1) >> s)) > kColdBins) s++;
  g.cold_shift = s;
  g.cold_nbins = (int)((ncold + (1ll << s) - 1) >> s);
  unsigned long long *cnt = nullptr;
  DI_CK(dmalloc(&cnt, kColdBins * 8));
  DI_CK(cudaMemsetAsync(cnt, 0, kColdBins * 8, g.stream));
  if (g.l > 0)
    k_cold_hist<<<g.num_sms * 8, 256, 0, g.stream>>>(g.col, g.l, g.cold_lo, s, cnt);
  std::vector<unsigned long long> hc(kColdBins);
  DI_CK(cudaMemcpyAsync(hc.data(), cnt, kColdBins * 8, cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  dfree(cnt);
  const int64_t slack = (int64_t)cycle_grid(g) * (kAsyncThreads / 32) * kColdChunk;
  std::vector<int64_t> off(kColdBins + 1, 0);
  for (int b = 0; b < g.cold_nbins; b++) {
    const int64_t cap = ((int64_t)hc[b] + slack + kColdChunk - 1) / kColdChunk * kColdChunk;
    if (cap >= (1ll << 31)) return DI_ENOMEM;   // positions inside a bin region are 32-bit
    off[b + 1] = off[b] + cap;
  }
  for (int b = g.cold_nbins; b < kColdBins; b++) off[b + 1] = off[b];
  const int64_t total = off[g.cold_nbins];
  DI_CK(dmalloc(&g.cold_rec, (size_t)total * sizeof(ColdRec)));
  DI_CK(dmalloc(&g.cold_fill, (size_t)(total / kColdChunk + 1) * 4));
  DI_CK(dmalloc(&g.cold_off, (kColdBins + 1) * 8));
  DI_CK(cudaMemcpyAsync(g.cold_off, off.data(), (kColdBins + 1) * 8, cudaMemcpyHostToDevice, g.stream));
  DI_CK(dmalloc(&g.cold_top, (kColdBins + 2) * 16 * 8));   // + ticket line + barrier line
  DI_CK(cudaMemsetAsync(g.cold_top, 0, (kColdBins + 2) * 16 * 8, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  return DI_OK;
}

// called by di_solve before any launch or capture (allocations are not capturable)
di_status prepare_cycle(Graph &g, bool async) {
  if (async && g.warm_count > 0) warm_init();   // (attributes are set outside any graph capture)
  if (async) {
    di_status cs = prepare_cold(g);
    if (cs != DI_OK) return cs;
  }
  if (g.cycle_times && !g.cyc_times)
    DI_CK(dmalloc(&g.cyc_times, (size_t)64 * kMaxSlices * 2 * sizeof(unsigned long long)));
  const int hot = hot_shift_of(g);
  if (hot >= 0 && !g.rep) {
    const size_t rep_bytes = ((size_t)kCopies * kRepl * kRepStride + kRepl) * sizeof(double);
    DI_CK(dmalloc(&g.rep, rep_bytes));
    DI_CK(cudaMemsetAsync(g.rep, 0, rep_bytes, g.stream));
    // hub items: hot rows longer than kHubMin, in kHubItem-link pieces (static: the CSR is)
    std::vector<int64_t> rp(hot + 1);
    DI_CK(cudaMemcpyAsync(rp.data(), g.row_ptr, (hot + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                          g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    std::vector<int64_t> items;
    for (int k = 0; k < hot; k++)
      if (rp[k + 1] - rp[k] > kHubMin)
        for (int64_t b = rp[k]; b < rp[k + 1]; b += kHubItem) {
          items.push_back(k);
          items.push_back(b);
          items.push_back(std::min(b + kHubItem, rp[k + 1]));
        }
    g.n_hub = (int)(items.size() / 3);
    if (g.n_hub > 0) {
      DI_CK(dmalloc(&g.hub_items, items.size() * sizeof(int64_t)));
      DI_CK(cudaMemcpyAsync(g.hub_items, items.data(), items.size() * sizeof(int64_t),
                            cudaMemcpyHostToDevice, g.stream));
      DI_CK(cudaStreamSynchronize(g.stream));
    }
  }
  return DI_OK;
}

static int cycle_grid(const Graph &g) {
  static const int occ = occupancy(k_cycle<false, false>, kAsyncThreads);  // once, thread-safe
  // option cycle_grid_div = k (experiments with emulated ranks on one GPU): 1/k of the grid per
  // rank, so the ranks' cycles run side by side at similar rates as they would on k GPUs
  return std::max(1, std::min(g.num_sms * occ, kMaxSlices) / std::max(1, g.grid_div));
}

// Warm accumulators a CTA of k_cycle<LOOPS, false, false, false, true> can hold without lowering the
// kernel's occupancy (the SM's shared memory split over its resident CTAs, less each CTA's static
// shared memory and the per-CTA reservation), in whole 256-id steps; the kernel's dynamic shared
// memory limit is raised to that once. Cached per instantiation (the device type is fixed).
template <bool LOOPS>
static int warm_cap() {
  static const int cap = [] {
    auto k = k_cycle<LOOPS, false, false, false, true>;
    int dev = 0, sm_bytes = 0, resv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sm_bytes, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return 0;
    const int occ = occupancy(k, kAsyncThreads);
    const int64_t per = (int64_t)sm_bytes / occ - resv - (int64_t)fa.sharedSizeBytes;
    const int c = per > 0 ? (int)((per / 8) & ~255ll) : 0;
    if (c > 0 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c * 8) != cudaSuccess)
      return 0;
    return c;
  }();
  return cap;
}

// the warm tier of k_cycle on this graph: a.warm warm-rank slots (0: off) + the hot ids
template <bool LOOPS>
static void set_warm(const Graph &g, SweepArgs &a) {
  a.warm = 0;
  a.warm_hot = (int32_t)g.hot_count;
  a.warm_shift = g.warm_shift;
  a.warm_flush = g.warm_flush;
  if (g.partitioned || g.warm_count <= 0) return;
  a.warm = (int)std::max<int64_t>(0, std::min<int64_t>(g.warm_count, warm_cap<LOOPS>() - g.hot_count));
}
static size_t warm_bytes(const SweepArgs &a) { return a.warm > 0 ? (size_t)(a.warm + a.warm_hot) * 8 : 0; }

// warm ranks k_cycle holds at full occupancy besides the hot ids (graph_build.cu: auto "warm";
// graphs with self-loops run the LOOPS instantiation, which holds fewer: set_warm clamps). Not
// with cold bins (graph_build.cu): only the non-COLD instantiations have a warm tier.
int warm_fit() { return std::max(0, warm_cap<false>() - kHotRanks); }

static void warm_init() {
  warm_cap<false>();
  warm_cap<true>();
}

// warps of k_cycle's grid (the cold regions reserve one chunk per warp of slack)
int64_t cycle_warps(const Graph &g) { return (int64_t)cycle_grid(g) * (kAsyncThreads / 32); }

// option cycle_times (diagnostic): per cycle, the spread of CTA start and end times (stderr)
void report_cycle_times(Graph &g, int64_t cycles) {
  if (!g.cyc_times || cycles <= 0) return;
  const int grid = cycle_grid(g);
  const int64_t nc = std::min<int64_t>(cycles, 64);
  std::vector<unsigned long long> t((size_t)nc * grid * 2);
  if (cudaMemcpy(t.data(), g.cyc_times, t.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  double span = 0, skew = 0, tail = 0, busy = 0;
  for (int64_t c = 0; c < nc; c++) {
    std::vector<double> st(grid), en(grid);
    for (int b = 0; b < grid; b++) {
      st[b] = (double)t[2 * (c * grid + b)];
      en[b] = (double)t[2 * (c * grid + b) + 1];
    }
    const double s0 = *std::min_element(st.begin(), st.end()), s1 = *std::max_element(st.begin(), st.end());
    std::vector<double> e2(en);
    std::sort(e2.begin(), e2.end());
    const double e1 = e2.back(), emed = e2[grid / 2];
    double b = 0;
    for (int k = 0; k < grid; k++) b += en[k] - st[k];
    span += e1 - s0;
    skew += s1 - s0;
    tail += e1 - emed;
    busy += b / grid;
  }
  fprintf(stderr, "[di cycle_times] %lld cycles, grid %d: span %.1f us, start skew %.1f us, tail (max - median end) %.1f us, mean CTA busy %.1f us\n",
          (long long)nc, grid, span / nc / 1e3, skew / nc / 1e3, tail / nc / 1e3, busy / nc / 1e3);
}

// di_test_cycle: one cycle of the select-and-take step on the current (F, H), recording (T, v)
void launch_cycle_test(Graph &g, double *rec_T, double *rec_v, int64_t *launches) {
  SweepArgs a = sweep_args(g, 1);
  a.ntiles = (g.n + kCycTile - 1) / kCycTile;
  a.hot_shift = g.rep ? hot_shift_of(g) : -1;
  a.rep = g.rep;
  a.times = nullptr;
  a.hub = nullptr;
  a.n_hub = 0;   // hub rows are recorded like the others (nothing is pushed)
  a.rec_T = rec_T;
  a.rec_v = rec_v;
  DistArgs x{};
  const int grid = cycle_grid(g);
  if (g.has_loops)
    k_cycle<true, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
  else
    k_cycle<false, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
  *launches += 1;
}

// k_cold_apply's grid: co-resident blocks only (its blocks wait for each other between bins)
static int cold_apply_grid(const Graph &g) {
  static const int occ = occupancy(k_cold_apply, 256);
  return g.num_sms * std::min(occ, 8);
}

void launch_cycle(Graph &g, int64_t *launches) {
  SweepArgs a = sweep_args(g, 0);
  a.long_lanes = g.long_lanes;
  const bool cold = g.cold_rec && !g.partitioned;
  if (cold) {
    a.cold_hot_tiles = (g.cold_lo + kCycTile - 1) / kCycTile;
    a.cold_lo = g.cold_lo;
    a.cold_shift = g.cold_shift;
    a.cold_nbins = g.cold_nbins;
    a.cold_rec = g.cold_rec;
    a.cold_off = g.cold_off;
    a.cold_top = g.cold_top;
    a.cold_fill = g.cold_fill;
  }
  a.ntiles = (g.n + kCycTile - 1) / kCycTile;
  const bool dist = g.partitioned;
  DistArgs x{};
  if (dist) x = dist_args(g);
  a.hot_shift = g.rep ? hot_shift_of(g) : -1;
  a.rep = g.rep;
  a.times = g.cyc_times;
  if (a.hot_shift >= 0) {
    a.hub = g.hub_items;
    a.n_hub = g.n_hub;
  }
  const int grid = cycle_grid(g);
  if (dist && g.dist_parts > 1 && g.cur_part >= 0) {   // this sweep: part cur_part of the cycle
    // (at most one part per tile: an empty part selects nothing and would trip the starvation
    //  guard into a threshold-0 sweep every other time)
    const int64_t T = a.ntiles, K = std::min<int64_t>(g.dist_parts, std::max<int64_t>(T, 1)),
                  p = g.cur_part % K;
    a.claim_lo = T * p / K;
    a.claim_hi = T * (p + 1) / K;
  }
  if (dist && g.cur_compact) {  // hot remote accumulator + cold records into the owners' inboxes
    x.ipar = g.cur_par;
    x.compact = 1;
    a.col = g.ccol;
    a.cold_hot_tiles = (g.rtier[g.rank] + kCycTile - 1) / kCycTile;
    if (g.has_loops)
      k_cycle<true, true, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    else
      k_cycle<false, true, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
  } else if (dist) {
    if (g.has_loops)
      k_cycle<true, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    else
      k_cycle<false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
  } else if (cold) {
    if (g.has_loops) {
      k_cycle<true, false, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    } else {
      k_cycle<false, false, false, true><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    }
    k_cold_apply<<<cold_apply_grid(g), 256, 0, g.stream>>>(g.F, g.cold_rec, g.cold_off, g.cold_top,
                                                           g.cold_fill, g.cold_nbins);
    *launches += 1;
  } else {
    if (g.has_loops) {
      set_warm<true>(g, a);
      if (a.warm > 0)
        k_cycle<true, false, false, false, true><<<grid, kAsyncThreads, warm_bytes(a), g.stream>>>(a, x);
      else
        k_cycle<true, false><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    } else {
      set_warm<false>(g, a);
      if (a.warm > 0)
        k_cycle<false, false, false, false, true><<<grid, kAsyncThreads, warm_bytes(a), g.stream>>>(a, x);
      else
        k_cycle<false, false><<<grid, kAsyncThreads, 0, g.stream>>>(a, x);
    }
  }
  *launches += 1;
}

}  // namespace di
