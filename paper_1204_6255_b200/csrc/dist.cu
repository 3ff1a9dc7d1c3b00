// dist.cu — D-iteration over a 1-D node partition, one rank per GPU.
//
// D-iteration is order-free (any sequence of diffusions keeps F = B + P.H - H), so a
// sweep splits into local diffusion plus one additive exchange of the fluid sent across the
// partition. Rank g owns nodes [lo, hi) (F, H, deg, kloop and the CSR rows of its sources with
// global column ids). One sweep on every rank:
//   1. k_select    — the single-GPU select/compact kernel on the owned nodes, global r_n.
//   2. k_push_dist — degree-binned push; a local target gets a RED into F, a remote target j a
//                    RED into the remote accumulator R[j] (global size, all-zero between
//                    sweeps). Its last block writes this rank's sweep sums.
//   3. k_compact_remote — one scan over R's remote segments: nonzero entries become (id, value)
//                    records in their owner's send segment, R back to zero, per-peer counts.
//   4. allreduce of the sweep sums; exchange of the per-peer counts (8 B per peer).
//   5. exchange of the (id int32, value fp64) records — 12 B per distinct (remote target, sweep)
//      pair, the algorithmic exchange of SURVEY §8(d), one send per peer.
//   6. k_apply_recv — F[j - lo] += value (RED: several peers may send the same j).
//   7. k_dist_finalize — the single-GPU finaliser on the global sums: every rank takes the same
//      stop / guard decision.
// With send/recv (step 5) the host reads the counts after step 4 (one synchronisation per sweep:
// NCCL needs the receive sizes on the host). With the peer-memory inboxes (the default) steps 3 and
// 5 are one kernel and the apply takes its counts from the gathered headers on the device, so the
// host enqueues batches of sweeps and reads the device state once per batch (the stop flag,
// counters and the dense/sparse choice), like the single-GPU loop. The collectives are NCCL
// (comm.cu), or the in-process group backend for emulated ranks on one GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "comm.cuh"
#include "sweep.cuh"

namespace di {
namespace {



// One target of one link: a RED into F (local) or into the remote accumulator R.
__device__ __forceinline__ void dist_add(const SweepArgs &a, const DistArgs &x, int32_t j, double v,
                                         bool valid, uint64_t fpol) {
  if (!valid) return;
  const int64_t jl = (int64_t)j - a.lo;
  if (jl >= 0 && jl < a.n)
    red_add_f64_hint(a.F + jl, v, fpol);
  else
    push_remote(x, j, v);
}

template <bool LOOPS>
__device__ __forceinline__ void dist_group(const SweepArgs &a, const DistArgs &x, int4 q, int64_t p0,
                                           int64_t beg, int64_t end, int32_t gi, double v,
                                           bool valid, uint64_t fpol) {
  const int32_t jj[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    const bool ok = valid && p >= beg && p < end && (!LOOPS || jj[c] != gi);
    dist_add(a, x, jj[c], v, ok, fpol);
  }
}

// The bins of k_push (diffusion.cu) with the local / remote routing of dist_add.
template <bool LOOPS>
__global__ void __launch_bounds__(kPushThreads) k_push_dist(const SweepArgs a, const DistArgs x) {
  __shared__ bool s_last;
  Scalars *sc = a.sc;
  if (sc->stop) return;
  const uint64_t pol = policy_evict_first();
  const uint64_t fpol = a.red_hint ? policy_evict_last() : policy_evict_normal();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kPushThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kPushThreads / 32) + (threadIdx.x >> 5);
  const int32_t *__restrict__ col = a.col;
  int64_t U[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) U[b] = (int64_t)sc->bin_fill[b][0];
  // bins C and W: warp per row (chunk)
  for (int b = BIN_C; b >= BIN_W; b--) {
    for (int64_t u = w; u < U[b]; u += W) {
      const Entry en = a.fr.ent[b][u];
      const int32_t gi = LOOPS ? (int32_t)(a.fr.id[b][u] + a.lo) : -1;
      const int64_t beg = (int64_t)(en.bl & kBegMask);
      const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
      const int64_t a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      const bool vpos = en.v > 0.0;
      for (int vb = 0; vb < nvec; vb += 32) {
        const int v0 = vb + lane;
        int4 q = make_int4(0, 0, 0, 0);
        if (v0 < nvec) q = ld_col4(col + a0 + 4 * (int64_t)v0, pol);
        dist_group<LOOPS>(a, x, q, a0 + 4 * (int64_t)v0, beg, end, gi, en.v, vpos && v0 < nvec, fpol);
      }
    }
  }
  // bin G: 8-lane group per row, 4 rows per warp step
  {
    const int sub = lane & 7;
    for (int64_t ub = 4 * w; ub < U[BIN_G]; ub += 4 * W) {
      const int64_t u = ub + (lane >> 3);
      const bool row = u < U[BIN_G];
      Entry en{0, 0.0};
      int32_t gi = -1;
      if (row) {
        en = a.fr.ent[BIN_G][u];
        if (LOOPS) gi = (int32_t)(a.fr.id[BIN_G][u] + a.lo);
      }
      const int64_t beg = (int64_t)(en.bl & kBegMask);
      const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
      const int64_t a0 = beg & ~3ll;
      const int nvec = row ? (int)((end - a0 + 3) >> 2) : 0;
      const bool vpos = en.v > 0.0;
      int4 q0 = make_int4(0, 0, 0, 0), q1 = make_int4(0, 0, 0, 0);
      if (sub < nvec) q0 = ld_col4(col + a0 + 4 * sub, pol);
      if (sub + 8 < nvec) q1 = ld_col4(col + a0 + 4 * (sub + 8), pol);
      dist_group<LOOPS>(a, x, q0, a0 + 4 * sub, beg, end, gi, en.v, vpos && sub < nvec, fpol);
      dist_group<LOOPS>(a, x, q1, a0 + 4 * (sub + 8), beg, end, gi, en.v, vpos && sub + 8 < nvec,
                        fpol);
    }
  }
  // bin T: one thread per row
  for (int64_t ub = 32 * w; ub < U[BIN_T]; ub += 32 * W) {
    const int64_t u = ub + lane;
    const bool row = u < U[BIN_T];
    Entry en{0, 0.0};
    int32_t gi = -1;
    if (row) {
      en = a.fr.ent[BIN_T][u];
      if (LOOPS) gi = (int32_t)(a.fr.id[BIN_T][u] + a.lo);
    }
    const int64_t beg = (int64_t)(en.bl & kBegMask);
    const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
    const int64_t a0 = beg & ~3ll;
    const int nvec = row ? (int)((end - a0 + 3) >> 2) : 0;
    const bool vpos = en.v > 0.0;
    int4 q0 = make_int4(0, 0, 0, 0), q1 = make_int4(0, 0, 0, 0), q2 = make_int4(0, 0, 0, 0);
    if (nvec > 0) q0 = ld_col4(col + a0, pol);
    if (nvec > 1) q1 = ld_col4(col + a0 + 4, pol);
    if (nvec > 2) q2 = ld_col4(col + a0 + 8, pol);
    dist_group<LOOPS>(a, x, q0, a0, beg, end, gi, en.v, vpos && nvec > 0, fpol);
    dist_group<LOOPS>(a, x, q1, a0 + 4, beg, end, gi, en.v, vpos && nvec > 1, fpol);
    dist_group<LOOPS>(a, x, q2, a0 + 8, beg, end, gi, en.v, vpos && nvec > 2, fpol);
  }
  // slices of the select partials; the last block: this rank's sweep sums and per-peer counts
  slice_partials(a, blockIdx.x, gridDim.x, kPushThreads);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const SweepSums s = reduce_partials(a, gridDim.x, kPushThreads);
  if (threadIdx.x == 0) {
    x.dsum[0] = s.q;
    x.dsum[1] = s.s;
    x.dsum[2] = s.e;
    x.dsum[3] = 0.0;
    x.isum[0] = s.sel;
    x.isum[1] = s.nd;
    x.isum[2] = s.lk;
    x.isum[3] = s.scanned;
    sc->ticket = 0;
  }
}

// Compaction of the remote accumulator (after the push, before the exchange): for every owner
// p != rank, the nonzero entries of R[b[p], b[p+1]) become 12-byte (id, value) records in p's
// send segment, and R returns to all-zero. Chunks of kCompChunk consecutive ids; each block
// reserves its chunk's records with one atomic (block scan for the positions), so the counter
// atomics are per chunk, not per entry. The last block publishes the per-peer counts into the
// sweep header and rewinds the counters. Record order inside a segment is the (free) reservation
// order; the receiver adds every record with a RED.
#ifndef DI_COMP_PER
#define DI_COMP_PER 4
#endif
#ifndef DI_COMP_BPS
#define DI_COMP_BPS 16
#endif
constexpr int kCompThreads = 256, kCompPer = DI_COMP_PER, kCompChunk = kCompThreads * kCompPer;
constexpr int kCompBlocksPerSM = DI_COMP_BPS;

// byte offset of the control lines in an inbox (after G segments of kRingSlots * icap records)
__host__ __device__ inline size_t ring_ctrl_offset(int world, int64_t icap) {
  return ((size_t)world * kRingSlots * (size_t)icap * 12 + 255) / 256 * 256;
}

__global__ void __launch_bounds__(kCompThreads) k_compact_remote(const Scalars *sc, DistArgs x) {
  __shared__ int s_w[kCompThreads / 32];
  __shared__ double s_sent[kCompThreads / 32];
  __shared__ unsigned long long s_base;
  __shared__ bool s_last;
  if (sc->stop) return;
  double sent = 0.0;   // ring mode: this thread's compacted fluid, over all its chunks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // chunk index space: owners in order, chunks of kCompChunk ids inside each (own range skipped)
  // (compact path: the segment of owner p is its hot prefix rt[p] in racc, L2-resident; else R's
  //  whole range of p)
  int64_t nchunks = 0;
  for (int p = 0; p < x.bd.world; p++)
    if (p != x.rank)
      nchunks += ((x.compact ? x.rt[p] : x.bd.b[p + 1] - x.bd.b[p]) + kCompChunk - 1) / kCompChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    int p = 0;
    int64_t cc = c;
    for (; p < x.bd.world; p++) {
      if (p == x.rank) continue;
      const int64_t k = ((x.compact ? x.rt[p] : x.bd.b[p + 1] - x.bd.b[p]) + kCompChunk - 1) / kCompChunk;
      if (cc < k) break;
      cc -= k;
    }
    // element k of this thread: id j0 + k * kCompThreads (a warp reads 32 consecutive doubles
    // per load: coalesced; the record order inside a segment is free)
    double *src = x.compact ? x.racc + x.hoff[p] - x.bd.b[p] : x.R;   // indexed by global id
    const int64_t j0 = x.bd.b[p] + cc * kCompChunk + (int64_t)threadIdx.x;
    const int64_t jend = x.bd.b[p] + (x.compact ? x.rt[p] : x.bd.b[p + 1] - x.bd.b[p]);
    double v[kCompPer];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kCompPer; k++) {
      const int64_t j = j0 + (int64_t)k * kCompThreads;
      v[k] = (j < jend) ? (x.compact ? __ldcg(src + j) : __ldcs(src + j)) : 0.0;
      cnt += (v[k] != 0.0) ? 1 : 0;
    }
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kCompThreads / 32; w++) {
      before += (w < warp) ? s_w[w] : 0;
      total += s_w[w];
    }
    if (threadIdx.x == 0)
      s_base = total ? atomicAdd(x.tcnt + 32 * p, (unsigned long long)total) : 0ull;
    __syncthreads();
    int64_t pos = (int64_t)s_base + before + incl - cnt;   // inside p's segment
    // fused exchange: p's inbox, segment of this rank, through peer memory (NVLink stores):
    // slot `ipar` (synchronous sweeps) or the ring from the published tail (DI_DIST_ASYNC);
    // otherwise p's segment of the local send buffer, moved by exchange()
    const int64_t seg = (int64_t)x.rank * kRingSlots * x.icap;
    const int64_t cap = (int64_t)kRingSlots * x.icap;
    int32_t *recs = x.p2p ? reinterpret_cast<int32_t *>(x.inbox[p]) +
                                3 * (seg + (x.ring ? 0 : (int64_t)x.ipar * x.icap))
                          : reinterpret_cast<int32_t *>(x.sval) + 3 * x.bd.b[p];
    const int64_t t0 = x.ring ? (int64_t)(x.tsent[p] % (unsigned long long)cap) : 0;  // ring start
#pragma unroll
    for (int k = 0; k < kCompPer; k++) {
      if (v[k] == 0.0) continue;
      const long long bits = __double_as_longlong(v[k]);
      int64_t at = pos;
      if (x.ring) {  // pos < one range <= cap: one wrap at most
        at = t0 + pos;
        if (at >= cap) at -= cap;
      }
      int32_t *r = recs + 3 * at;
      r[0] = (int32_t)(j0 + (int64_t)k * kCompThreads);
      r[1] = (int32_t)(bits & 0xffffffffll);
      r[2] = (int32_t)(bits >> 32);
      src[j0 + (int64_t)k * kCompThreads] = 0.0;
      sent += v[k];
      pos++;
    }
    __syncthreads();  // s_w / s_base reused by the next chunk
  }
  if (x.ring) {  // fluid that left this rank (the local r estimate, DI_DIST_ASYNC): one atomic
    sent = warp_sum(sent);   // per block (same-address fp64 atomics serialise in one L2 slice)
    if (lane == 0) s_sent[warp] = sent;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kCompThreads / 32; w++) t += s_sent[w];
      if (t != 0.0) atomicAdd(x.sent, t);
    }
  }
  // the last block: per-peer counts into the header, counters rewound. Ring mode: the block's
  // records (ordered before thread 0 by the barrier) reach the peers before the ticket, hence
  // before the last block publishes the tails; synchronous sweeps: the kernel's completion
  // orders them before the collective that hands the counts over
  __syncthreads();
  if (threadIdx.x == 0) {
    if (x.ring)
      __threadfence_system();
    else
      __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned int *>(x.tcnt + 32 * x.bd.world), 1u) ==
             gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < x.bd.world) {
    volatile unsigned long long *cn = x.tcnt + 32 * threadIdx.x;
    const unsigned long long c = *cn;
    x.sendcnt[threadIdx.x] = (threadIdx.x == x.rank) ? 0 : (int64_t)c;
    *cn = 0ull;
    if (x.compact) {  // cold records reserved in the owner's inbox this cycle (k_cycle)
      volatile unsigned long long *ct = x.ctop + 16 * threadIdx.x;
      x.coldcnt[threadIdx.x] = (threadIdx.x == x.rank) ? 0 : (int64_t)*ct;
      *ct = 0ull;
    } else if (x.coldcnt) {
      x.coldcnt[threadIdx.x] = 0;
    }
    if (x.ring && threadIdx.x != x.rank) {  // publish the new tail in the owner's control line
      const unsigned long long t = x.tsent[threadIdx.x] + c;
      x.tsent[threadIdx.x] = t;
      unsigned long long *ctl = reinterpret_cast<unsigned long long *>(
          x.inbox[threadIdx.x] + ring_ctrl_offset(x.bd.world, x.icap) + 256 * (size_t)x.rank);
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ctl), "l"(t) : "memory");
    }
  }
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned int *>(x.tcnt + 32 * x.bd.world) = 0u;
}

__global__ void k_apply_recv(double *__restrict__ F, int64_t lo, const int32_t *__restrict__ rec,
                             int64_t m) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t *r = rec + 3 * k;
    const double v = __longlong_as_double(((long long)(uint32_t)r[1]) | ((long long)r[2] << 32));
    red_add_f64(F + ((int64_t)r[0] - lo), v);
  }
}

// fused exchange, receiving side: the records every peer wrote into this rank's inbox segment
// (parity, peer); the counts come from the gathered sweep headers (device-resident)
__global__ void k_apply_inbox(double *__restrict__ F, int64_t lo, const char *__restrict__ inbox,
                              int64_t icap, int ipar, const int64_t *__restrict__ ghdr, int world,
                              int me, const Scalars *sc, int64_t ccap, size_t cold_off0,
                              size_t fill_off0) {
  if (sc->stop) return;   // batched loop: a sweep after convergence (stale headers) does nothing
  const int hw = hdr_words(world);
  for (int q = 0; q < world; q++) {   // compact path: the cold records sender q wrote (16 B)
    if (q == me || ccap == 0) continue;
    const int64_t mc = ghdr[(int64_t)q * hw + 8 + world + me];
    const ColdRec *rec = reinterpret_cast<const ColdRec *>(inbox + cold_off0) + (2 * q + ipar) * ccap;
    const int32_t *fill = reinterpret_cast<const int32_t *>(inbox + fill_off0) +
                          (2 * q + ipar) * (ccap / kColdChunk);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < mc;
         k += (int64_t)gridDim.x * blockDim.x) {
      if ((int)(k % kColdChunk) >= fill[k / kColdChunk]) continue;
      const int4 r = *reinterpret_cast<const int4 *>(rec + k);
      red_add_f64(F + r.x, __hiloint2double(r.w, r.z));   // (cold records carry the local id)
    }
  }
  for (int q = 0; q < world; q++) {
    if (q == me) continue;
    const int64_t m = ghdr[(int64_t)q * hw + 8 + me];
    const int32_t *rec = reinterpret_cast<const int32_t *>(inbox) +
                         3 * ((int64_t)q * kRingSlots * icap + (int64_t)ipar * icap);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
      const int32_t *r = rec + 3 * k;
      const double v = __longlong_as_double(((long long)(uint32_t)r[1]) | ((long long)r[2] << 32));
      red_add_f64(F + ((int64_t)r[0] - lo), v);
    }
  }
}

// DI_DIST_ASYNC receiving side, step 1: the tails the peers published (acquire: their records
// are visible after it); every block of the apply then uses the same snapshot
__global__ void k_ring_snap(const char *inbox, int world, int64_t icap, int me,
                            unsigned long long *snap) {
  const int q = threadIdx.x;
  if (q >= world || q == me) return;
  const unsigned long long *ctl = reinterpret_cast<const unsigned long long *>(
      inbox + ring_ctrl_offset(world, icap) + 256 * (size_t)q);
  unsigned long long t;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(t) : "l"(ctl) : "memory");
  snap[q] = t;
}

// step 2: records [head, snap) of every peer's ring into F (RED), the fluid summed into *applied
__global__ void k_ring_apply(double *__restrict__ F, int64_t lo, const char *__restrict__ inbox,
                             int world, int64_t icap, int me, const unsigned long long *snap,
                             const unsigned long long *head, double *applied) {
  const int64_t cap = (int64_t)kRingSlots * icap;
  double acc = 0.0;
  for (int q = 0; q < world; q++) {
    if (q == me) continue;
    const int64_t h = (int64_t)head[q], m = (int64_t)snap[q] - h;
    const int32_t *seg = reinterpret_cast<const int32_t *>(inbox) + 3 * ((int64_t)q * cap);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
      const int32_t *r = seg + 3 * ((h + k) % cap);
      const double v = __longlong_as_double(((long long)(uint32_t)r[1]) | ((long long)r[2] << 32));
      red_add_f64(F + ((int64_t)r[0] - lo), v);
      acc += v;
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(applied, acc);
}

// step 3: the ring heads advance to the snapshot
__global__ void k_ring_advance(int world, int me, const unsigned long long *snap,
                               unsigned long long *head) {
  const int q = threadIdx.x;
  if (q < world && q != me) head[q] = snap[q];
}

// DI_DIST_ASYNC: this rank's cycle effect on its own fluid, r_loc <- r_loc - taken + pushed -
// sent + applied, and the r of the next cycle's threshold (reading R8 in DESIGN.md): the global
// r of the last meeting times (r_loc + sent) / r_loc at that meeting. Measured on emulated ranks
// (tools/exp/dist_async.py): the rule on the rank's own part, r_loc / L_loc, or the decay
// without the sent fluid, over-diffuse (C4 at G = 2: 64 and 49 eq-iter vs 44.3 with this one,
// 44.75 for synchronous cycles); counters; the starvation guard
__global__ void k_ring_finalize(const SweepArgs a, const DistArgs x, double *rs) {
  if (threadIdx.x != 0) return;
  Scalars *sc = a.sc;
  const double taken = x.dsum[3], pushed = x.dsum[1], e = x.dsum[2];
  const double sent = rs[0];
  const double r_loc = rs[2] - taken + pushed - sent + rs[1];
  rs[0] = 0.0;
  rs[1] = 0.0;
  rs[2] = r_loc;
  // the global r of the last meeting, scaled by this rank's decay since; the fluid it just sent
  // still counts (it left for the peers, it did not leave the system)
  const double rl = (r_loc > 0.0 ? r_loc : 0.0) + sent;
  sc->r = (rs[3] > 0.0) ? rs[4] * rl / rs[3] : rs[4];
  sc->e = sc->e + e;
  sc->sweeps = sc->sweeps + 1;
  sc->selected_total = sc->selected_total + x.isum[0];
  sc->selected_nd_total = sc->selected_nd_total + x.isum[1];
  sc->links_total = sc->links_total + x.isum[2];
  sc->scanned_total = sc->scanned_total + a.n;
  const int starving = (x.isum[0] == 0 && sc->variant == DI_SOP) ? 1 : 0;
  if (starving) sc->guards = sc->guards + 1;
  sc->guard = starving;
}

// meeting: r_loc = r_loc at the meeting = this rank's exact sum F (resid); r = the global sum
__global__ void k_ring_meet(Scalars *sc, const double *global, double *rs) {
  rs[2] = sc->resid;
  rs[3] = sc->resid;
  rs[4] = *global;
  sc->r = *global;
}

// dense fallback: this rank's slice of the reduced accumulators into F
__global__ void k_apply_dense(double *__restrict__ F, const double *__restrict__ recv, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double v = recv[k];
    if (v != 0.0) F[k] += v;
  }
}

// the single-GPU finaliser on the sums of the gathered headers (rank order: every rank computes
// the same values bit for bit)
__global__ void k_dist_finalize(const SweepArgs a, const int64_t *ghdr, int world, int async,
                                int me, int p2p) {
  if (threadIdx.x != 0 || a.sc->stop) return;
  const int hw = hdr_words(world);
  {  // exchange counters (entries this rank sent; every rank's entries of this sweep)
    int64_t mine = 0, all = 0, cold = 0;
    for (int p = 0; p < world; p++)
      for (int q = 0; q < world; q++)
        if (p != q) {
          const int64_t c = ghdr[(int64_t)p * hw + 8 + q];
          all += c;
          if (p == me) {
            mine += c;
            cold += ghdr[(int64_t)p * hw + 8 + world + q];
          }
        }
    volatile Scalars *vs = a.sc;
    vs->x_entries = vs->x_entries + mine;
    vs->x_cold = vs->x_cold + cold;
    vs->x_lists_last = all;
    if (p2p) vs->x_p2p = vs->x_p2p + 1;
  }
  double d[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t c[4] = {0, 0, 0, 0};
  for (int p = 0; p < world; p++) {
    const int64_t *h = ghdr + (int64_t)p * hw;
    for (int k = 0; k < 4; k++) d[k] += __longlong_as_double(h[k]);
    for (int k = 0; k < 4; k++) c[k] += h[4 + k];
  }
  // the asynchronous cycle reports the fluid it took from F (d[3]) instead of the fluid it
  // left: r_{c+1} = r_c - taken + pushed, i.e. q = r_c - taken for apply_sweep's q + s
  const double q = async ? __dsub_rn(a.sc->r, d[3]) : d[0];
  SweepSums s{q, d[1], d[2], 0.0, c[0], c[1], c[2], c[3]};
  apply_sweep(a, s);
}

__global__ void k_set_r(Scalars *sc, const double *sum, int set_r) {
  sc->resid = *sum;
  if (set_r) sc->r = *sum;
}

__global__ void k_copy_resid(const Scalars *sc, double *out) { *out = sc->resid; }

int grid_of(int64_t n, int sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
}


// global sum F (exact local tree sum, then the allreduce); set_r: also r = that sum
di_status global_sum_F(Graph &g, int set_r, int64_t *launches) {
  launch_reduce_F(g, launches);
  double *scratch = reinterpret_cast<double *>(g.hdr + hdr_words(g.world));
  k_copy_resid<<<1, 1, 0, g.stream>>>(g.sc, scratch);
  di_status s = g.comm->allreduce_f64(scratch, 1, g.stream);
  if (s != DI_OK) return s;
  k_set_r<<<1, 1, 0, g.stream>>>(g.sc, scratch, set_r);
  *launches += 2;
  return DI_OK;
}

// links of this rank whose target is a cold remote target (j outside [lo, hi) and not in its
// owner's hot prefix), per owner: the capacity of the cold regions of the inboxes
__global__ void k_cold_remote_count(const int32_t *__restrict__ col, int64_t L, DistBounds bd,
                                    int me, const int64_t *rt, unsigned long long *cnt) {
  __shared__ unsigned int h[kMaxWorld];
  if (threadIdx.x < kMaxWorld) h[threadIdx.x] = 0u;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[k];
    int p = 0;
    while (p + 1 < bd.world && j >= bd.b[p + 1]) p++;
    if (p != me && j - bd.b[p] >= rt[p]) atomicAdd(&h[p], 1u);
  }
  __syncthreads();
  if (threadIdx.x < bd.world && h[threadIdx.x]) atomicAdd(cnt + threadIdx.x, (unsigned long long)h[threadIdx.x]);
}

// The compact path's column encoding (one pass at upload): a local target j becomes j - lo, a
// hot remote target (within the first rt[p] ids of its owner's range p) becomes n + hoff[p] +
// (j - b[p]) — its accumulator slot after the n local ids — and a colder remote target n + R + j
// (R = sum of rt): the push then needs two compares, and an owner lookup only for cold targets.
__global__ void k_encode_col(const int32_t *__restrict__ col, int64_t L, int64_t lo, int64_t n,
                             DistBounds bd, const int64_t *rt, const int64_t *hoff, int64_t R,
                             int64_t W, int32_t *__restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[k];
    int64_t e;
    if (j >= lo && j < lo + n) {
      e = j - lo;
    } else {
      int p = 0;
      while (p + 1 < bd.world && j >= bd.b[p + 1]) p++;
      const int64_t off = j - bd.b[p];
      e = off < rt[p] ? n + hoff[p] + off : n + R + p * W + off;   // (owner p, its local id)
    }
    out[k] = (int32_t)e;
  }
}

}  // namespace

// the global-size remote accumulator and the send/recv buffers: only the bulk partitioned sweep,
// the asynchronous multi-GPU cycles (rings), the send/recv and dense exchanges use them
di_status ensure_R(Graph &g) {
  if (g.R_ready) return DI_OK;
  const int64_t N = g.n_global;
  const int G = g.world;
  DI_CK(dmalloc(&g.R, (size_t)N * 8));
  DI_CK(dmemset(g.R, 0, (size_t)N * 8));
  DI_CK(dmalloc(&g.sval, (size_t)N * 12));   // send records, segment p at record b[p]
  const size_t cap = (size_t)std::max<int64_t>(1, (int64_t)(G - 1) * g.n);
  DI_CK(dmalloc(&g.rid, cap * 12));          // received records
  g.R_ready = true;
  return DI_OK;
}

di_status alloc_dist(Graph &g) {
  const int G = g.world;
  DI_CK(dmalloc(&g.tcnt, (size_t)(G + 1) * 32 * 8));   // + the compaction's block ticket
  DI_CK(dmemset(g.tcnt, 0, (size_t)(G + 1) * 32 * 8));
  const size_t hw = (size_t)hdr_words(G);
  DI_CK(dmalloc(&g.hdr, 8 * 8 + hw * 8));   // +8 words: global_sum_F's scratch after the header
  DI_CK(dmemset(g.hdr, 0, 8 * 8 + hw * 8));
  DI_CK(dmalloc(&g.ghdr, (size_t)G * hw * 8));
  DI_CK(cudaMallocHost(&g.ghdr_h, (size_t)G * hw * 8));
  g.dsum = reinterpret_cast<double *>(g.hdr);
  g.isum = g.hdr + 4;
  g.sendcnt = g.hdr + 8;
  // compact remote path: accumulator of the hot remote targets, cold-record counters, and the
  // capacity of the inboxes' cold regions (the largest count of any sender -> owner pair plus
  // one chunk per warp of the sender's cycle grid; allgathered: the same on every rank)
  int64_t rsum = 0;
  for (int p = 0; p < G; p++) rsum += g.rtier[p];
  const bool compact_ok = g.reordered && g.remote_compact && rsum > 0;
  g.ccap = 0;
  if (compact_ok) {
    DI_CK(dmalloc(&g.racc, (size_t)rsum * 8));
    DI_CK(dmemset(g.racc, 0, (size_t)rsum * 8));
    DI_CK(dmalloc(&g.ctop, (size_t)2 * kMaxWorld * 16 * 8));
    DI_CK(dmemset(g.ctop, 0, (size_t)2 * kMaxWorld * 16 * 8));
    int64_t *rtd = nullptr;
    unsigned long long *cnt = nullptr;
    DI_CK(dmalloc(&rtd, kMaxWorld * 8));
    DI_CK(dmalloc(&cnt, (size_t)G * G * 8));
    DI_CK(cudaMemcpyAsync(rtd, g.rtier, kMaxWorld * 8, cudaMemcpyHostToDevice, g.stream));
    DI_CK(cudaMemsetAsync(cnt, 0, (size_t)G * G * 8, g.stream));
    if (g.l > 0)
      k_cold_remote_count<<<g.num_sms * 8, 256, 0, g.stream>>>(g.col, g.l, g.bounds, g.rank, rtd,
                                                                cnt + (size_t)g.rank * G);
    std::vector<int64_t> mine(G);
    DI_CK(cudaMemcpyAsync(mine.data(), cnt + (size_t)g.rank * G, (size_t)G * 8, cudaMemcpyDeviceToHost,
                          g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    const int64_t slack = cycle_warps(g) * (int64_t)kColdChunk;
    for (int p = 0; p < G; p++) mine[p] += slack;
    DI_CK(cudaMemcpy(cnt + (size_t)g.rank * G, mine.data(), (size_t)G * 8, cudaMemcpyHostToDevice));
    di_status s0 = g.comm->allgather(cnt + (size_t)g.rank * G, cnt, (size_t)G * 8, g.stream);
    if (s0 != DI_OK) return s0;
    std::vector<int64_t> all((size_t)G * G);
    DI_CK(cudaMemcpyAsync(all.data(), cnt, (size_t)G * G * 8, cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    dfree(rtd);
    dfree(cnt);
    int64_t mx = kColdChunk;
    for (int q = 0; q < G; q++)
      for (int p = 0; p < G; p++)
        if (p != q) mx = std::max<int64_t>(mx, all[(size_t)q * G + p]);
    g.ccap = (mx + kColdChunk - 1) / kColdChunk * kColdChunk;
    // the encoded columns: local ids, hot remote slots, then owner windows of W = the largest
    // range (a cold target's owner is one multiply away in k_cycle, no table lookup); the
    // encoding must fit int32 on every rank: W + R + G W < 2^31
    int64_t W = 1;
    for (int p = 0; p < G; p++) W = std::max<int64_t>(W, g.bounds.b[p + 1] - g.bounds.b[p]);
    g.cwin = W;
    if ((double)W + (double)rsum + (double)G * (double)W >= 2147483647.0) {
      g.ccap = 0;   // no compact path on this graph
    } else {
      int64_t hoff[kMaxWorld + 1];
      hoff[0] = 0;
      for (int p = 0; p < G; p++) hoff[p + 1] = hoff[p] + g.rtier[p];
      int64_t *dv = nullptr;
      DI_CK(dmalloc(&dv, 2 * (kMaxWorld + 1) * 8));
      DI_CK(cudaMemcpyAsync(dv, g.rtier, kMaxWorld * 8, cudaMemcpyHostToDevice, g.stream));
      DI_CK(cudaMemcpyAsync(dv + kMaxWorld + 1, hoff, (kMaxWorld + 1) * 8, cudaMemcpyHostToDevice,
                            g.stream));
      DI_CK(dmalloc(&g.ccol, (size_t)(g.l + 8) * 4));
      DI_CK(cudaMemsetAsync(g.ccol + g.l, 0, 8 * 4, g.stream));
      if (g.l > 0)
        k_encode_col<<<g.num_sms * 8, 256, 0, g.stream>>>(g.col, g.l, g.lo, g.n, g.bounds, dv,
                                                           dv + kMaxWorld + 1, rsum, W, g.ccol);
      DI_CK(cudaStreamSynchronize(g.stream));
      dfree(dv);
    }
  }
  // fused exchange: a double-buffered inbox of G segments of (largest range) records per rank,
  // written by the peers' compaction kernels through peer memory (collective; every rank agrees
  // on the outcome, else all fall back to exchange())
  g.p2p = false;
  g.inbox.clear();
  // (option p2p = 0 disables it; p2p_force = 1 creates it on one rank too, which exercises the
  // symmetric-memory calls with nothing to send)
  const bool want = G > 1 || g.p2p_force == 1;
  if (want && g.p2p_opt != 0) {
    int64_t mx = 1;
    for (int p = 0; p < G; p++) mx = std::max<int64_t>(mx, g.bounds.b[p + 1] - g.bounds.b[p]);
    g.icap = mx;
    // [G segments of kRingSlots x icap 12-B records][G control lines][cold regions: per sender 2
    // parities x ccap 16-B records][their chunk fills: per sender 2 x ccap / kColdChunk int32]
    g.cold_off0 = (ring_ctrl_offset(G, mx) + (size_t)256 * G + 255) / 256 * 256;
    g.fill_off0 = (g.cold_off0 + (size_t)G * 2 * (size_t)g.ccap * sizeof(ColdRec) + 255) / 256 * 256;
    const size_t ibytes = g.fill_off0 + (size_t)G * 2 * (size_t)(g.ccap / kColdChunk) * 4 + 256;
    std::vector<char *> peers;
    di_status s = g.comm->make_inbox(ibytes, &peers);
    if (s == DI_OK &&  // ring tails start at 0 (the allreduce below orders it before any use)
        cudaMemset(peers[g.rank] + ring_ctrl_offset(G, mx), 0, (size_t)256 * G) != cudaSuccess)
      s = DI_ECUDA;
    int64_t *flag = reinterpret_cast<int64_t *>(g.ghdr);   // scratch before the first sweep
    const int64_t bad = (s == DI_OK) ? 0 : 1;
    DI_CK(cudaMemcpy(flag, &bad, 8, cudaMemcpyHostToDevice));
    di_status s2 = g.comm->allreduce_i64(flag, 1, g.stream);
    if (s2 != DI_OK) return s2;
    int64_t nbad = 0;
    DI_CK(cudaMemcpy(&nbad, flag, 8, cudaMemcpyDeviceToHost));
    if (nbad == 0) {
      g.inbox = peers;
      g.p2p = true;
      DI_CK(dmalloc(&g.ring, 3 * kMaxWorld * 8 + 8 * 8));
      DI_CK(dmemset(g.ring, 0, 3 * kMaxWorld * 8 + 8 * 8));
    } else {
      g.comm->free_inbox();
    }
  }
  return DI_OK;
}

void free_dist(Graph &g) {
  void *p[] = {g.R, g.sval, g.tcnt, g.hdr, g.ghdr, g.rid, g.ring, g.racc, g.ctop, g.ccol};
  for (void *q : p)
    if (q) dfree(q);
  if (g.ghdr_h) cudaFreeHost(g.ghdr_h);
  if (g.comm) g.comm->free_inbox();
  g.inbox.clear();
  g.p2p = false;
  delete g.comm;
  g.comm = nullptr;
}

di_status dist_residual(Graph &g, double *l1) {
  int64_t launches = 0;
  di_status s = global_sum_F(g, 0, &launches);
  if (s != DI_OK) return s;
  DI_CK(cudaMemcpyAsync(l1, g.hdr + hdr_words(g.world), 8, cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  return DI_OK;
}

// DI_DIST_ASYNC: asynchronous cycles across ranks. Every rank runs its own
// cycles (k_cycle<DIST>) back to back; the fluid for remote targets goes through the peer-memory
// rings (k_compact_remote in ring mode appends and publishes the tail; each rank drains its
// rings at the start of every cycle), so no collective separates two cycles. The ranks meet
// every kRingSlots cycles — which bounds what a sender can have in flight to one ring — to drain
// everything, take the exact global sum F and decide convergence; between meetings a rank's
// DI-SOP threshold scales the last global r by its own fluid's decay (reading R8).
di_status solve_dist_async(Graph &g, double d, const double *B, double tol, int variant,
                           int64_t max_sweeps, uint32_t flags, di_stats *st) {
  const int G = g.world, me = g.rank;
  if (!g.p2p || !g.ring) {
    set_error("di_solve: DI_DIST_ASYNC needs the peer-memory inboxes (option p2p)");
    return DI_EINVAL;
  }
  const bool resume = flags & DI_RESUME;
  const int paper = (flags & DI_PAPER_ERROR) ? 1 : 0;
  int64_t launches = 0;
  cudaEvent_t t0, t1;
  DI_CK(cudaEventCreate(&t0));
  DI_CK(cudaEventCreate(&t1));
  {
    Scalars &s = *g.sc_host;
    const uint32_t epoch = s.epoch ? s.epoch : 1;
    memset(&s, 0, sizeof(Scalars));
    s.epoch = epoch;
    s.e = 0.0;   // this rank's absorption; the global e is summed at the meetings (g.e_global)
    s.d = d;
    s.tol = tol;
    s.variant = variant;
    s.paper_err = paper;
    s.alpha = g.alpha;
    s.mode = MODE_PUSH;
  }
  double e_global = resume ? g.e_global : 0.0;
  g.cur_compact = 0;
  {
    di_status rs = ensure_R(g);   // the rings compact the global-size accumulator
    if (rs != DI_OK) return rs;
  }
  DI_CK(cudaEventRecord(t0, g.stream));
  DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  DI_CK(cudaMemsetAsync(g.R, 0, (size_t)g.n_global * 8, g.stream));
  DI_CK(cudaMemsetAsync(g.tcnt, 0, (size_t)(G + 1) * 32 * 8, g.stream));
  if (!resume) launch_init(g, B, d, &launches);
  unsigned long long *tsent = g.ring, *head = g.ring + kMaxWorld, *snap = g.ring + 2 * kMaxWorld;
  double *rs = reinterpret_cast<double *>(g.ring + 3 * kMaxWorld);
  double *scratch = reinterpret_cast<double *>(g.hdr + hdr_words(g.world));
  unsigned long long sent0[kMaxWorld];   // ring tails at the start: entries sent = difference
  DI_CK(cudaMemcpyAsync(sent0, tsent, sizeof(sent0), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaMemsetAsync(rs, 0, 8 * 8, g.stream));
  const char *mine = g.inbox[me];
  auto drain = [&]() {
    k_ring_snap<<<1, 32, 0, g.stream>>>(mine, G, g.icap, me, snap);
    k_ring_apply<<<g.num_sms * 4, 256, 0, g.stream>>>(g.F, g.lo, mine, G, g.icap, me, snap, head,
                                                      rs + 1);
    k_ring_advance<<<1, 32, 0, g.stream>>>(G, me, snap, head);
    launches += 3;
  };
  // a meeting: everyone's cycles and their ring appends are complete (collective 1, which also
  // sums the dangling absorption), every ring is drained, the exact global sum F (collective 2)
  auto meet = [&](double *r_out) -> di_status {
    DI_CK(cudaMemcpyAsync(scratch, &g.sc->e, 8, cudaMemcpyDeviceToDevice, g.stream));
    di_status s = g.comm->allreduce_f64(scratch, 1, g.stream);
    if (s != DI_OK) return s;
    double e_sum = 0.0;
    DI_CK(cudaMemcpyAsync(&e_sum, scratch, 8, cudaMemcpyDeviceToHost, g.stream));
    drain();
    launch_reduce_F(g, &launches);   // this rank's exact sum F -> sc->resid
    k_copy_resid<<<1, 1, 0, g.stream>>>(g.sc, scratch + 1);
    if ((s = g.comm->allreduce_f64(scratch + 1, 1, g.stream)) != DI_OK) return s;
    k_ring_meet<<<1, 1, 0, g.stream>>>(g.sc, scratch + 1, rs);
    launches += 2;
    DI_CK(cudaMemcpyAsync(r_out, scratch + 1, 8, cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    g.e_cycle = e_sum;
    return DI_OK;
  };
  auto err_of = [&](double r, double e) { return paper ? r / (1.0 - d - d * e) : r; };
  double r_glob = 0.0;
  di_status s = meet(&r_glob);
  if (s != DI_OK) return s;
  bool converged = err_of(r_glob, e_global + g.e_cycle) <= tol;
  const SweepArgs a = sweep_args(g, 0);
  DistArgs x = dist_args(g);
  x.p2p = 1;
  x.ring = 1;
  int64_t launched = 0, meetings = 1;
  const bool prof = flags & DI_PROFILE;   // events around every cycle kernel (roofline)
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (prof) {
    DI_CK(cudaEventCreate(&pe0));
    DI_CK(cudaEventCreate(&pe1));
  }
  double push_ms = 0.0;
  int64_t push_launches = 0;
  while (!converged && launched < max_sweeps) {
    const int64_t k_end = std::min<int64_t>(max_sweeps, launched + kRingSlots);
    for (; launched < k_end; launched++) {
      drain();                       // what the peers sent so far
      if (prof) DI_CK(cudaEventRecord(pe0, g.stream));
      launch_cycle(g, &launches);    // this rank's asynchronous cycle (R7) with r from rs
      if (prof) {
        DI_CK(cudaEventRecord(pe1, g.stream));
        DI_CK(cudaEventSynchronize(pe1));
        float c_ms = 0.f;
        cudaEventElapsedTime(&c_ms, pe0, pe1);
        push_ms += c_ms;
        push_launches++;
      }
      k_compact_remote<<<g.num_sms * kCompBlocksPerSM, kCompThreads, 0, g.stream>>>(g.sc, x);
      k_ring_finalize<<<1, 32, 0, g.stream>>>(a, x, rs);
      launches += 2;
    }
    if ((s = meet(&r_glob)) != DI_OK) return s;
    meetings++;
    converged = err_of(r_glob, e_global + g.e_cycle) <= tol;
  }
  // global counters (every rank reports the same totals)
  DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  {
    int64_t *cnt = reinterpret_cast<int64_t *>(scratch + 2);
    const int64_t h[5] = {g.sc_host->selected_total, g.sc_host->selected_nd_total,
                          g.sc_host->links_total, g.sc_host->scanned_total, g.sc_host->guards};
    DI_CK(cudaMemcpyAsync(cnt, h, sizeof(h), cudaMemcpyHostToDevice, g.stream));
    if ((s = g.comm->allreduce_i64(cnt, 5, g.stream)) != DI_OK) return s;
    int64_t tot[5];
    DI_CK(cudaMemcpyAsync(tot, cnt, sizeof(tot), cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    Scalars &c = *g.sc_host;
    c.selected_total = tot[0];
    c.selected_nd_total = tot[1];
    c.links_total = tot[2];
    c.scanned_total = tot[3];
    c.guards = tot[4];
    c.resid = r_glob;
    c.r = r_glob;
    c.e = e_global + g.e_cycle;
    c.sweeps = launched;
    DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  }
  g.e_global = g.sc_host->e;
  if (pe0) cudaEventDestroy(pe0);
  if (pe1) cudaEventDestroy(pe1);
  unsigned long long sent1[kMaxWorld];
  DI_CK(cudaMemcpyAsync(sent1, tsent, sizeof(sent1), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaEventRecord(t1, g.stream));
  DI_CK(cudaEventSynchronize(t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  DI_CK(cudaGetLastError());
  g.solved = true;
  g.last_d = d;
  g.log_n = 0;
  if (st) {
    const Scalars &c = *g.sc_host;
    memset(st, 0, sizeof(*st));
    st->sweeps = c.sweeps;
    st->selected_total = c.selected_total;
    st->link_diffusions = c.links_total;
    st->starvation_fallbacks = c.guards;
    st->nodes_scanned = c.scanned_total;
    st->gpu_launches = launches;
    st->residual_l1 = c.resid;
    st->dangling_absorbed = c.e;
    st->equivalent_iterations = g.l_global > 0 ? (double)c.links_total / (double)g.l_global : 0.0;
    st->solve_ms = ms;
    st->counted_bytes = 12.0 * c.scanned_total + 40.0 * c.selected_total + 20.0 * c.links_total;
    st->push_bytes = 16.0 * c.selected_nd_total + 20.0 * c.links_total;
    st->error_estimate = c.resid / (1.0 - d - d * c.e);
    st->converged = converged ? 1 : 0;
    st->variant = variant;
    st->p2p_exchanges = launched;
    st->meetings = meetings;
    st->push_ms = push_ms;
    st->push_launches = push_launches;
    int64_t ent = 0;
    for (int p = 0; p < G; p++) ent += (p == me) ? 0 : (int64_t)(sent1[p] - sent0[p]);
    st->exchange_entries = ent;
    st->exchange_bytes = 12.0 * (double)ent;
  }
  return converged ? DI_OK : DI_NOT_CONVERGED;
}

di_status solve_dist(Graph &g, double d, const double *B, double tol, int variant,
                     int64_t max_sweeps, uint32_t flags, di_stats *st) {
  if (flags & DI_DIST_ASYNC) {
    if (!(flags & DI_ASYNC))
    {  // F2 runs R7 cycles on every rank
      set_error("di_solve: DI_DIST_ASYNC runs asynchronous cycles (add DI_ASYNC)");
      return DI_EINVAL;
    }
    return solve_dist_async(g, d, B, tol, variant, max_sweeps, flags, st);
  }
  const int G = g.world, me = g.rank;
  const bool resume = flags & DI_RESUME;
  const bool async = flags & DI_ASYNC;
  const int paper = (flags & DI_PAPER_ERROR) ? 1 : 0;
  int64_t launches = 0;
  cudaEvent_t t0, t1;
  DI_CK(cudaEventCreate(&t0));
  DI_CK(cudaEventCreate(&t1));
  {
    Scalars &s = *g.sc_host;
    const uint32_t epoch = s.epoch ? s.epoch : 1;
    const double e_prev = s.e;
    memset(&s, 0, sizeof(Scalars));
    s.epoch = epoch;
    s.e = resume ? e_prev : 0.0;
    s.d = d;
    s.tol = tol;
    s.variant = variant;
    s.paper_err = paper;
    s.alpha = g.alpha;
    s.trace = (flags & DI_TRACE) ? 1 : 0;
    s.mode = MODE_PUSH;
  }
  // the compact remote path (hot remote accumulator + cold records into the owners' inboxes):
  // asynchronous cycles through peer memory; everything else uses the global-size accumulator
  const bool p2p = g.p2p && !(flags & DI_XCHG_NOP2P);
  const bool compact = async && p2p && g.racc && g.ccap > 0 && !(flags & DI_XCHG_DENSE);
  if (!compact) {
    di_status rs = ensure_R(g);
    if (rs != DI_OK) return rs;
  }
  DI_CK(cudaEventRecord(t0, g.stream));
  DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  if (compact) {
    int64_t rsum = 0;
    for (int p = 0; p < G; p++) rsum += g.rtier[p];
    DI_CK(cudaMemsetAsync(g.racc, 0, (size_t)rsum * 8, g.stream));
    DI_CK(cudaMemsetAsync(g.ctop, 0, (size_t)2 * kMaxWorld * 16 * 8, g.stream));
  } else {
    DI_CK(cudaMemsetAsync(g.R, 0, (size_t)g.n_global * 8, g.stream));
  }
  DI_CK(cudaMemsetAsync(g.tcnt, 0, (size_t)(G + 1) * 32 * 8, g.stream));
  g.cur_compact = compact ? 1 : 0;
  di_status s = DI_OK;
  if (!resume) {
    launch_init(g, B, d, &launches);  // F = B (local slice), H = 0; local sum
  }
  s = global_sum_F(g, 1, &launches);
  if (s != DI_OK) return s;
  DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  auto err_of = [&](double r, double e) { return paper ? r / (1.0 - d - d * e) : r; };
  bool converged = err_of(g.sc_host->r, g.sc_host->e) <= tol;
  const SweepArgs a = sweep_args(g, 0);
  DistArgs x = dist_args(g);
  x.p2p = p2p ? 1 : 0;
  x.compact = compact ? 1 : 0;
  int par = 0;   // inbox parity of the current sweep
  int occ = 0;
  if (g.has_loops)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push_dist<true>, kPushThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push_dist<false>, kPushThreads, 0);
  occ = std::max(1, occ);
  std::vector<const void *> sb(G);
  std::vector<void *> rb(G);
  std::vector<size_t> s12(G), r12(G);
  const size_t hw = (size_t)hdr_words(G);
  double xbytes = 0.0, xdense = 0.0;
  int64_t ndense = 0, np2p = 0;   // (entries sent are counted on the device: Scalars::x_entries)
  // exchange choice: sparse lists unless the last sparse sweep's lists
  // (12 B per entry, all ranks) outweighed the dense reduction (8 B per remote node per rank);
  // after kDenseRun dense sweeps one sparse sweep measures the lists again
  constexpr int kDenseRun = 4;
  const bool force_dense = (flags & DI_XCHG_DENSE) && G > 1;
  const bool force_sparse = (flags & DI_XCHG_SPARSE) || G == 1 || compact;
  int64_t last_lists = -1;
  int dense_run = 0;
  int64_t launched = 0;
  const bool prof = flags & DI_PROFILE;
  cudaEvent_t pe[4] = {nullptr, nullptr, nullptr, nullptr};
  if (prof)
    for (auto &e : pe) DI_CK(cudaEventCreate(&e));
  double push_ms = 0.0, select_ms = 0.0, xchg_ms = 0.0;
  int64_t push_launches = 0;
  int64_t batch = 4;
  int64_t part_ctr = 0;   // option dist_parts: the part of the rank's cycle each sweep takes
  double r_prev = g.sc_host->r;
  while (!converged && launched < max_sweeps) {
    // ---- batched sweeps through peer memory: no host synchronisation inside a batch
    const bool batched = p2p && !prof && !force_dense &&
                         !(!force_sparse && last_lists >= 0 &&
                           12.0 * (double)last_lists > 8.0 * (double)(G - 1) * (double)g.n_global);
    if (batched) {
      const int64_t k = std::min<int64_t>(batch, max_sweeps - launched);
      const int64_t sw0 = g.sc_host->sweeps;
      for (int64_t j = 0; j < k; j++) {
        if (!async) launch_select(g, 0, &launches);
        g.cur_par = par;   // the cold regions written by this cycle
        g.cur_part = (int)(part_ctr++ % g.dist_parts);
        if (async)
          launch_cycle(g, &launches);
        else if (g.has_loops)
          k_push_dist<true><<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a, x);
        else
          k_push_dist<false><<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a, x);
        x.ipar = par;
        k_compact_remote<<<g.num_sms * kCompBlocksPerSM, kCompThreads, 0, g.stream>>>(g.sc, x);
        if ((s = g.comm->allgather(g.hdr, g.ghdr, (size_t)hw * 8, g.stream)) != DI_OK) return s;
        k_apply_inbox<<<g.num_sms * 4, 256, 0, g.stream>>>(g.F, g.lo, g.inbox[me], g.icap, par,
                                                          g.ghdr, G, me, g.sc, compact ? g.ccap : 0,
                                                          g.cold_off0, g.fill_off0);
        k_dist_finalize<<<1, 32, 0, g.stream>>>(a, g.ghdr, G, async ? 1 : 0, me, 1);
        launches += 4;
        par ^= 1;
      }
      launched += k;
      DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
      DI_CK(cudaStreamSynchronize(g.stream));   // once per batch
      DI_CK(cudaGetLastError());
      const int64_t real = g.sc_host->sweeps - sw0;
      last_lists = g.sc_host->x_lists_last;
      if (g.sc_host->stop) {
        launched = g.sc_host->sweeps;
      } else if (launched < max_sweeps) {
        // next batch: the sweeps left predicted from the decay of r (as on one GPU)
        const double r_now = g.sc_host->r;
        int64_t next = 8;
        if (real > 0 && r_now > 0.0 && r_prev > r_now) {
          const double rate = std::pow(r_now / r_prev, 1.0 / (double)real);
          const double target = paper ? tol * (1.0 - d) : tol;
          if (rate < 1.0 && rate > 0.0)
            next = (int64_t)std::ceil(std::max(1.0, std::log(target / r_now) / std::log(rate)));
        }
        batch = std::max<int64_t>(1, std::min<int64_t>(next, 32));
        r_prev = r_now;
        continue;
      }
    }
    while (!batched && launched < max_sweeps) {
      if (prof) DI_CK(cudaEventRecord(pe[0], g.stream));
      if (!async) launch_select(g, 0, &launches);
      if (prof) DI_CK(cudaEventRecord(pe[1], g.stream));
      g.cur_par = par;
      g.cur_part = (int)(part_ctr++ % g.dist_parts);
      if (async)
        launch_cycle(g, &launches);   // the asynchronous cycle on this rank's range (R7)
      else if (g.has_loops)
        k_push_dist<true><<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a, x);
      else
        k_push_dist<false><<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a, x);
      if (prof) DI_CK(cudaEventRecord(pe[2], g.stream));
      const bool dense =
          force_dense ||
          (!force_sparse && dense_run < kDenseRun && last_lists >= 0 &&
           12.0 * (double)last_lists > 8.0 * (double)(G - 1) * (double)g.n_global);
      if (dense)  // no lists: the header's per-peer counts are zero
        DI_CK(cudaMemsetAsync(g.sendcnt, 0, (size_t)G * 8, g.stream));
      else {
        x.ipar = par;
        k_compact_remote<<<g.num_sms * kCompBlocksPerSM, kCompThreads, 0, g.stream>>>(g.sc, x);
      }
      launches += 2;
      launched++;
      // one collective for the sums and the per-peer counts of every rank
      if ((s = g.comm->allgather(g.hdr, g.ghdr, (size_t)hw * 8, g.stream)) != DI_OK) return s;
      DI_CK(cudaMemcpyAsync(g.ghdr_h, g.ghdr, (size_t)G * hw * 8, cudaMemcpyDeviceToHost,
                            g.stream));
      DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
      DI_CK(cudaStreamSynchronize(g.stream));
      if (g.sc_host->stop) {  // the previous sweep converged: this one was a no-op on every rank
        launched--;
        break;
      }
      if (prof) {
        float a01 = 0.f, a12 = 0.f;
        cudaEventElapsedTime(&a01, pe[0], pe[1]);
        cudaEventElapsedTime(&a12, pe[1], pe[2]);
        select_ms += a01;
        push_ms += a12;
        push_launches++;
        DI_CK(cudaEventRecord(pe[3], g.stream));
      }
      int64_t off = 0;
      if (dense) {  // per-owner reduction of R, then R's remote segments back to zero
        double *recv = reinterpret_cast<double *>(g.rid);
        if ((s = g.comm->reduce_segments(g.R, recv, g.bounds.b, g.stream)) != DI_OK) return s;
        k_apply_dense<<<grid_of(g.n, g.num_sms), 256, 0, g.stream>>>(g.F, recv, g.n);
        const int64_t b0 = g.bounds.b[me], b1 = g.bounds.b[me + 1];
        if (b0 > 0) DI_CK(cudaMemsetAsync(g.R, 0, (size_t)b0 * 8, g.stream));
        if (b1 < g.n_global)
          DI_CK(cudaMemsetAsync(g.R + b1, 0, (size_t)(g.n_global - b1) * 8, g.stream));
        launches++;
        xdense += 8.0 * (double)(g.n_global - g.n);
        ndense++;
        dense_run++;
      } else {
        last_lists = 0;
        for (int p = 0; p < G; p++)
          for (int q = 0; q < G; q++) last_lists += (p == q) ? 0 : g.ghdr_h[(size_t)p * hw + 8 + q];
        dense_run = 0;
      }
      if (!dense && p2p) {  // the records are already in the owners' inboxes: apply ours
        k_apply_inbox<<<g.num_sms * 4, 256, 0, g.stream>>>(g.F, g.lo, g.inbox[me], g.icap, par,
                                                          g.ghdr, G, me, g.sc, compact ? g.ccap : 0,
                                                          g.cold_off0, g.fill_off0);
        launches++;
        par ^= 1;
        np2p++;
      }
      for (int p = 0; p < G && !dense && !p2p; p++) {
        const int64_t ns = (p == me) ? 0 : g.ghdr_h[(size_t)me * hw + 8 + p];
        const int64_t nr = (p == me) ? 0 : g.ghdr_h[(size_t)p * hw + 8 + me];
        sb[p] = reinterpret_cast<const char *>(g.sval) + (size_t)12 * g.bounds.b[p];
        s12[p] = (size_t)ns * 12;
        rb[p] = reinterpret_cast<char *>(g.rid) + (size_t)12 * off;
        r12[p] = (size_t)nr * 12;
        off += nr;
      }
      if (!dense && !p2p &&
          (s = g.comm->exchange(sb.data(), s12.data(), rb.data(), r12.data(), g.stream)) != DI_OK)
        return s;
      if (off > 0) {
        k_apply_recv<<<grid_of(off, g.num_sms), 256, 0, g.stream>>>(g.F, g.lo, g.rid, off);
        launches++;
      }
      k_dist_finalize<<<1, 32, 0, g.stream>>>(a, g.ghdr, G, async ? 1 : 0, me, 0);
      launches++;
      if (prof) {  // exchange of the lists + apply (the counts exchange is in the sync above)
        DI_CK(cudaEventRecord(pe[0], g.stream));
        DI_CK(cudaEventSynchronize(pe[0]));
        float a30 = 0.f;
        cudaEventElapsedTime(&a30, pe[3], pe[0]);
        xchg_ms += a30;
      }
      // the device decided; its stop flag is read back with the next sweep's counts
    }
    // exact global residual (deterministic on each rank, summed by the collective)
    if ((s = global_sum_F(g, 0, &launches)) != DI_OK) return s;
    DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    converged = err_of(g.sc_host->resid, g.sc_host->e) <= tol;
    if (converged || !g.sc_host->stop) break;
    // the q + s prediction said converged but the exact sum disagrees by rounding: continue
    const int32_t zero = 0;
    DI_CK(cudaMemcpyAsync(&g.sc->stop, &zero, 4, cudaMemcpyHostToDevice, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    g.sc_host->stop = 0;
  }
  g.cur_part = -1;   // (other callers of launch_cycle take whole cycles)
  if (launched == 0 && !converged) {
    if ((s = global_sum_F(g, 0, &launches)) != DI_OK) return s;
    DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
  }
  for (auto e : pe)
    if (e) cudaEventDestroy(e);
  DI_CK(cudaEventRecord(t1, g.stream));
  DI_CK(cudaEventSynchronize(t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  DI_CK(cudaGetLastError());
  g.solved = true;
  g.last_d = d;
  g.log_n = std::min<int64_t>(g.sc_host->sweeps, kLogCap);
  if (st) {
    const Scalars &c = *g.sc_host;
    memset(st, 0, sizeof(*st));
    st->sweeps = c.sweeps;
    st->selected_total = c.selected_total;
    st->link_diffusions = c.links_total;
    st->starvation_fallbacks = c.guards;
    st->nodes_scanned = c.scanned_total;
    st->gpu_launches = launches;
    st->residual_l1 = c.resid;
    st->dangling_absorbed = c.e;
    st->equivalent_iterations = g.l_global > 0 ? (double)c.links_total / (double)g.l_global : 0.0;
    st->solve_ms = ms;
    st->counted_bytes = 12.0 * c.scanned_total + 40.0 * c.selected_total + 20.0 * c.links_total;
    st->push_bytes = 16.0 * c.selected_nd_total + 20.0 * c.links_total;
    st->error_estimate = c.resid / (1.0 - d - d * c.e);
    st->converged = converged ? 1 : 0;
    st->variant = variant;
    xbytes = 12.0 * (double)c.x_entries + 16.0 * (double)c.x_cold + xdense;
    st->exchange_bytes = xbytes;
    st->dense_exchanges = ndense;
    st->p2p_exchanges = np2p + c.x_p2p;
    st->exchange_entries = c.x_entries;
    st->exchange_cold = c.x_cold;
    st->push_ms = push_ms;
    st->select_ms = select_ms;
    st->push_launches = push_launches;
    st->exchange_ms = xchg_ms;
  }
  return converged ? DI_OK : DI_NOT_CONVERGED;
}

}  // namespace di
