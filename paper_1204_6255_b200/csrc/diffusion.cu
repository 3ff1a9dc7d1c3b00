// diffusion.cu — the D-iteration hot path on sm_100a.
//
// One bulk-synchronous sweep n (R1) is two kernels:
//   k_select  (a2+a3+a4): for every node i, test F_i against the DI-SOP threshold
//             (r_n/L)*#out_i (literal order, reading G4) or 0 (DI-CYC);
//             for selected i: T_i = F_i, or F_i*#out_i/(#out_i - k_i*d) with k_i self-loops
//             (reading G6); H_i += T_i; F_i = 0; dangling: e += T_i
//             (P:266-267); else emit the row (first link, #out_i, v_i = T_i*d/#out_i) into the
//             degree bin of #out_i. A tile reserves its range of each bin with one atomicAdd
//             and writes its entries in ascending node order (no inter-block waiting). The
//             same pass writes per-tile partial sums of q = sum of unselected F and
//             s = sum T_i*d*(#out_i-k_i)/#out_i, so r_{n+1} = q + s is known when the sweep
//             ends (a2) without another pass over F.
//   k_push    (a5): F_j += v_i for every link i -> j, j != i, fp64 RED atomics,
//             degree-binned: hub chunks and W rows one warp each, G rows one 8-lane group,
//             T rows one thread. Its last block finalises the sweep (a6): fixed-order
//             reduction of the partials, r_{n+1}, the stop test, the starvation guard (G5).
// All solve parameters live in device memory (Scalars), so the sweep is a fixed pair of
// launches with constant arguments (CUDA-graph capturable); once `stop` is set both kernels
// return immediately, so the host can enqueue sweeps ahead without reading anything back.
#include <vector>

#include "di_common.cuh"
#include "kern_util.cuh"
#include "sweep.cuh"

namespace di {
namespace {

// ------------------------------------------------------------------ init (a1)
__global__ void k_init(double *__restrict__ F, double *__restrict__ H, const double *__restrict__ B,
                       double b0, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    F[i] = B ? B[i] : b0;
    H[i] = 0.0;
  }
}

// --------------------------------------------- deterministic sum of a vector
// Fixed grid, fixed per-thread striding, fixed tree: bitwise reproducible for a given n.
// mode 1: also set r = sum (sweep threshold at solve start).
__global__ void __launch_bounds__(kRedThreads) k_reduce(const double *__restrict__ x, int64_t n,
                                                        double *__restrict__ partials,
                                                        Scalars *sc, int mode) {
  __shared__ double s_w[kRedThreads / 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kRedThreads)
    a += x[i];
  a = warp_sum(a);
  if (lane == 0) s_w[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; w++) t += s_w[w];
    partials[blockIdx.x] = t;
    __threadfence();
    s_last = atomicAdd(&sc->red_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  a = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kRedThreads) a += __ldcg(partials + b);
  a = warp_sum(a);
  if (lane == 0) s_w[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRedThreads / 32; w++) t += s_w[w];
    sc->resid = t;
    if (mode == 1) sc->r = t;
    sc->red_ticket = 0;
  }
}

int reduce_grid(int64_t n, int sms) {
  int64_t g = (n + kRedThreads * 8 - 1) / (kRedThreads * 8);
  if (g > (int64_t)sms * 4) g = (int64_t)sms * 4;
  if (g < 1) g = 1;
  return (int)g;
}

// -------------------------------------------------------- select + compact (a2-a4)
// One tile = kSelTile consecutive nodes; thread t owns kSelItems consecutive nodes.
template <bool LOOPS>
__global__ void __launch_bounds__(kSelThreads, 3) k_select(const SweepArgs a) {
  constexpr int NW = kSelThreads / 32;
  __shared__ int s_wcnt[NW][kBins];
  __shared__ double s_red[NW][4];
  __shared__ int64_t s_links[NW];
  __shared__ int s_sel[NW], s_selnd[NW];
  __shared__ unsigned long long s_res[kBins];

  Scalars *sc = a.sc;
  if (!a.test_mode && sc->stop) return;
  const int64_t tile = a.t0 + blockIdx.x;   // block-ordered sweeps scan tiles [t0, t1)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double r = sc->r;
  const double d = sc->d;
  const bool cyc = (sc->variant == DI_CYC) || sc->guard;
  const int mode = sc->mode;
  const bool emit = mode != MODE_PULL, dense = mode != MODE_PUSH;
  double t = (a.L_total > 0.0) ? r / a.L_total : 0.0;  // r/L once (G3, G4)
  if (sc->alpha != 1.0) t = __dmul_rn(t, sc->alpha);  // F4 threshold scale (1 = the paper's rule)
  const int64_t base = tile * (int64_t)kSelTile + (int64_t)threadIdx.x * kSelItems;
  const bool full = base + kSelItems <= a.n;

  double f[kSelItems];
  int o[kSelItems];
  int kl[kSelItems];
  int64_t rb[kSelItems];  // row extents row_ptr[i] (the push's first link); o_i = rb_{i+1} - rb_i
  // One round trip: F and row_ptr stream in together (coalesced); #out_i comes from the row
  // extent instead of a separate deg read, so no second dependent load is needed for the
  // selected rows' first link.
  if (full) {
    const double2 *F2 = reinterpret_cast<const double2 *>(a.F + base);
    const longlong2 *R2 = reinterpret_cast<const longlong2 *>(a.row_ptr + base);
    int64_t rnext;
#pragma unroll
    for (int j = 0; j < kSelItems / 2; j++) {
      const double2 x = F2[j];
      f[2 * j] = x.x;
      f[2 * j + 1] = x.y;
      const longlong2 r = R2[j];
      rb[2 * j] = r.x;
      rb[2 * j + 1] = r.y;
    }
    rnext = a.row_ptr[base + kSelItems];
#pragma unroll
    for (int j = 0; j < kSelItems; j++) o[j] = (int)((j + 1 < kSelItems ? rb[j + 1] : rnext) - rb[j]);
    if (LOOPS) {
      const int4 *K4 = reinterpret_cast<const int4 *>(a.kloop + base);
#pragma unroll
      for (int j = 0; j < kSelItems / 4; j++) {
        const int4 x = K4[j];
        kl[4 * j] = x.x;
        kl[4 * j + 1] = x.y;
        kl[4 * j + 2] = x.z;
        kl[4 * j + 3] = x.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kSelItems; j++) {
      const int64_t i = base + j;
      f[j] = (i < a.n) ? a.F[i] : 0.0;
      rb[j] = (i < a.n) ? a.row_ptr[i] : 0;
      o[j] = (i < a.n) ? (int)(a.row_ptr[i + 1] - rb[j]) : 0;
      if (LOOPS) kl[j] = (i < a.n) ? a.kloop[i] : 0;
    }
  }
  if (!LOOPS) {
#pragma unroll
    for (int j = 0; j < kSelItems; j++) kl[j] = 0;
  }

  // ---- pass 1: the selection test (P:258 / P:298) and the bin counts
  uint32_t selmask = 0, dangmask = 0;
  int cnt[kBins] = {0, 0, 0, 0};
  double q = 0.0, tk = 0.0;   // fluid left unselected / taken from F by the selection
#pragma unroll
  for (int j = 0; j < kSelItems; j++) {
    const int64_t i = base + j;
    if (i >= a.n) continue;
    const double thr = cyc ? 0.0 : __dmul_rn(t, (double)o[j]);  // (r/L)*out[i]
    if (f[j] > thr) {                                             // strict '>'
      tk = __dadd_rn(tk, f[j]);
      if (o[j] == 0) {
        dangmask |= 1u << j;
      } else {
        selmask |= 1u << j;
        const int b = bin_of(o[j]);
        const int inc = (b == BIN_C) ? (o[j] + kChunk - 1) / kChunk : 1;
#pragma unroll
        for (int bb = 0; bb < kBins; bb++) cnt[bb] += (bb == b) ? inc : 0;  // no local memory
      }
    } else {
      q = __dadd_rn(q, f[j]);
    }
  }
  // ---- pass 2a: move the fluid of selected nodes into H. H_i += T is a RED: the
  //      L2 adds in fp64 round-to-nearest exactly as a load/add/store would (H_i is touched by
  //      this thread only), without a dependent load.
  const uint32_t anysel = selmask | dangmask;
  double v[kSelItems];
#pragma unroll
  for (int j = 0; j < kSelItems; j++) v[j] = 0.0;
  double s = 0.0, e = 0.0;
  int64_t links = 0;
  int nsel = 0, nsel_nd = 0;
  if (anysel) {
#pragma unroll
    for (int j = 0; j < kSelItems; j++) {
      if (!(anysel & (1u << j))) continue;
      const int64_t i = base + j;
      const double od = (double)o[j];
      double T = f[j];
      if (LOOPS && kl[j] > 0)                           // P:259-263 with k copies (G6)
        T = __ddiv_rn(__dmul_rn(f[j], od), __dsub_rn(od, __dmul_rn((double)kl[j], d)));
      red_add_f64(a.H + i, T);
      a.F[i] = 0.0;
      nsel++;
      if (o[j] == 0) {
        e = __dadd_rn(e, T);
      } else {
        v[j] = __ddiv_rn(__dmul_rn(T, d), od);          // sent = transit*d/out[i]
        s = __dadd_rn(s, __dmul_rn(v[j], (double)(o[j] - kl[j])));  // fluid leaving i
        links += o[j];
        nsel_nd++;
      }
    }
  }
  // pull variant: dense S (v_i for diffused non-dangling nodes, 0 elsewhere), read by k_pull
  if (dense) {
    if (full) {
      double2 *S2 = reinterpret_cast<double2 *>(a.S + base);
#pragma unroll
      for (int j = 0; j < kSelItems / 2; j++)
        S2[j] = make_double2((selmask >> (2 * j) & 1u) ? v[2 * j] : 0.0,
                             (selmask >> (2 * j + 1) & 1u) ? v[2 * j + 1] : 0.0);
    } else {
#pragma unroll
      for (int j = 0; j < kSelItems; j++)
        if (base + j < a.n) a.S[base + j] = (selmask >> j & 1u) ? v[j] : 0.0;
    }
  }

  // ---- block-wide exclusive scan of the 4 bin counts, one reservation per bin
  int incl[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) {
    int x = cnt[b];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    incl[b] = x;
    if (lane == 31) s_wcnt[warp][b] = x;
  }
  __syncthreads();
  int pos[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) {
    int we = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      const int c = s_wcnt[w][b];
      we += (w < warp) ? c : 0;
      tot += c;
    }
    pos[b] = we + incl[b] - cnt[b];
    if (threadIdx.x == b)
      s_res[b] = (tot && emit) ? atomicAdd(&sc->bin_fill[b][0], (unsigned long long)tot) : 0ull;
  }
  __syncthreads();

  // ---- pass 2b: emit the rows into the reserved ranges, ascending node id inside each bin
  if (selmask && emit) {
    int64_t slot[kBins];
#pragma unroll
    for (int b = 0; b < kBins; b++) slot[b] = (int64_t)s_res[b] + pos[b];
#pragma unroll
    for (int j = 0; j < kSelItems; j++) {
      if (!(selmask & (1u << j))) continue;
      const int32_t i = (int32_t)(base + j);
      const int b = bin_of(o[j]);
      if (b != BIN_C) {
        Entry en;
        en.bl = (uint64_t)rb[j] | ((uint64_t)o[j] << kLenShift);
        en.v = v[j];
#pragma unroll
        for (int bb = 0; bb < BIN_C; bb++) {
          if (bb == b) {
            a.fr.ent[bb][slot[bb]] = en;
            a.fr.id[bb][slot[bb]] = i;
            slot[bb]++;
          }
        }
      } else {
        const int nch = (o[j] + kChunk - 1) / kChunk;
        for (int c = 0; c < nch; c++) {
          const int len = min(kChunk, o[j] - c * kChunk);
          Entry en;
          en.bl = (uint64_t)(rb[j] + (int64_t)c * kChunk) | ((uint64_t)len << kLenShift);
          en.v = v[j];
          a.fr.ent[BIN_C][slot[BIN_C] + c] = en;
          a.fr.id[BIN_C][slot[BIN_C] + c] = i;
        }
        slot[BIN_C] += nch;
      }
    }
  }

  // ---- block partials (fixed order), reduced by the sweep finaliser
  q = warp_sum(q);
  s = warp_sum(s);
  e = warp_sum(e);
  tk = warp_sum(tk);
  links = warp_sum(links);
  nsel = warp_sum(nsel);
  nsel_nd = warp_sum(nsel_nd);
  if (lane == 0) {
    s_red[warp][0] = q;
    s_red[warp][1] = s;
    s_red[warp][2] = e;
    s_red[warp][3] = tk;
    s_links[warp] = links;
    s_sel[warp] = nsel;
    s_selnd[warp] = nsel_nd;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tq = 0.0, ts = 0.0, te = 0.0, tt = 0.0;
    int64_t tl = 0;
    int tsel = 0, tnd = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      tq += s_red[w][0];
      ts += s_red[w][1];
      te += s_red[w][2];
      tt += s_red[w][3];
      tl += s_links[w];
      tsel += s_sel[w];
      tnd += s_selnd[w];
    }
    reinterpret_cast<double2 *>(a.partials)[2 * tile] = make_double2(tq, ts);
    reinterpret_cast<double2 *>(a.partials)[2 * tile + 1] = make_double2(te, tt);
    reinterpret_cast<longlong2 *>(a.ipartials)[2 * tile] = make_longlong2(tsel, tnd);
    if (mode == MODE_AUTO && tl) atomicAdd(&sc->fill_links[0], (unsigned long long)tl);
    reinterpret_cast<longlong2 *>(a.ipartials)[2 * tile + 1] = make_longlong2(tl, 0);
  }
}

__global__ void __launch_bounds__(kPushThreads) k_finalize(const SweepArgs a) {
  slice_partials(a, 0, 1, kPushThreads);
  __syncthreads();
  __threadfence();
  finalize_sweep(a, 1, kPushThreads);
}

// Static capacity of every bin (rows, or chunks for C) from the degrees: per select tile in
// shared memory, then one atomic per tile and bin into the totals.
__global__ void __launch_bounds__(kSelThreads) k_tile_caps(const int32_t *__restrict__ deg,
                                                           int64_t n,
                                                           unsigned long long *__restrict__ tot) {
  __shared__ int s_c[kBins];
  if (threadIdx.x < kBins) s_c[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  int c[kBins] = {0, 0, 0, 0};
  for (int k = threadIdx.x; k < kSelTile; k += kSelThreads) {
    const int64_t i = base + k;
    if (i >= n) break;
    const int o = deg[i];
    if (o == 0) continue;
    const int b = bin_of(o);
    const int inc = (b == BIN_C) ? (o + kChunk - 1) / kChunk : 1;
#pragma unroll
    for (int bb = 0; bb < kBins; bb++) c[bb] += (bb == b) ? inc : 0;
  }
#pragma unroll
  for (int b = 0; b < kBins; b++) {
    const int x = warp_sum(c[b]);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&s_c[b], x);
  }
  __syncthreads();
  if (threadIdx.x < kBins && s_c[threadIdx.x])
    atomicAdd(tot + threadIdx.x, (unsigned long long)s_c[threadIdx.x]);
}

// ------------------------------------------------------------------ push (a5)
// rows of > kBinG links (bins W and C): one warp per row. Entries are dealt round-robin
// (u = w, w + W, ...): rows of similar size cluster in a bin (tile order, hubs first after the
// relabelling), so contiguous ranges would load-imbalance. Warp-uniform broadcast entry loads,
// prefetched one ahead; 2 int4 groups (8 links) per lane in flight.
template <bool LOOPS>
__device__ __forceinline__ void push_rows_warp(const SweepArgs &a, int b, int64_t w, int64_t W,
                                               int64_t U, int lane, uint64_t pol, uint64_t fpol) {
  if (w >= U) return;
  const Entry *__restrict__ ent = a.fr.ent[b];
  const int32_t *__restrict__ col = a.col;
  double *__restrict__ F = a.F;
  double *__restrict__ rep = a.rep;   // replicated hot accumulators (j < hot_lim)
  const int32_t hot_lim = a.hot_shift > 0 ? a.hot_shift : 0;
  const int copy = (int)(((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) % kRepCopies);
  Entry nx = ent[w];
  for (int64_t u = w; u < U; u += W) {
    const Entry en = nx;
    if (u + W < U) nx = ent[u + W];
    const int32_t gi = LOOPS ? (int32_t)(a.fr.id[b][u] + a.lo) : -1;
    const int64_t beg = (int64_t)(en.bl & kBegMask);
    const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
    const int64_t a0 = beg & ~3ll;
    const int nvec = (int)((end - a0 + 3) >> 2);
    for (int vb = 0; vb < nvec; vb += 64) {
      const int v0 = vb + lane, v1 = vb + 32 + lane;
      int4 x0 = make_int4(0, 0, 0, 0), x1 = make_int4(0, 0, 0, 0);
      if (v0 < nvec) x0 = ld_col4(col + a0 + 4 * (int64_t)v0, pol);
      if (v1 < nvec) x1 = ld_col4(col + a0 + 4 * (int64_t)v1, pol);
      if (v0 < nvec) red_group<LOOPS>(F, rep, hot_lim, copy, x0, a0 + 4 * (int64_t)v0, beg, end, gi, en.v, fpol);
      if (v1 < nvec) red_group<LOOPS>(F, rep, hot_lim, copy, x1, a0 + 4 * (int64_t)v1, beg, end, gi, en.v, fpol);
    }
  }
}

template <bool LOOPS, int MINB>
__global__ void __launch_bounds__(kPushThreads, MINB) k_push(const SweepArgs a) {
  __shared__ bool s_last;
  Scalars *sc = a.sc;
  if (sc->stop) return;
  const int mode = sc->mode;
  if (mode == MODE_AUTO && (int64_t)sc->fill_links[0] > sc->pull_thr) return;  // k_pull's sweep
  const uint64_t pol = policy_evict_first();
  const uint64_t fpol = a.red_hint ? policy_evict_last() : policy_evict_normal();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kPushThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kPushThreads / 32) + (threadIdx.x >> 5);
  const int32_t *__restrict__ col = a.col;
  double *__restrict__ F = a.F;
  double *__restrict__ rep = a.rep;   // replicated hot accumulators (j < hot_lim)
  const int32_t hot_lim = a.hot_shift > 0 ? a.hot_shift : 0;
  const int copy = (int)(((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) % kRepCopies);
  int64_t U[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) U[b] = (int64_t)sc->bin_fill[b][0];
  // ---- bins C (hub chunks) and W: warp per row
  push_rows_warp<LOOPS>(a, BIN_C, w, W, U[BIN_C], lane, pol, fpol);
  push_rows_warp<LOOPS>(a, BIN_W, w, W, U[BIN_W], lane, pol, fpol);
  // ---- bin G (9..32 links): 8-lane group per row, 4 rows per warp step; <= 9 int4 groups
  {
    const int sub = lane & 7;
    const int64_t u1 = U[BIN_G];
    for (int64_t u = 4 * w + (lane >> 3); u < u1; u += 4 * W) {
      const Entry en = a.fr.ent[BIN_G][u];
      const int32_t gi = LOOPS ? (int32_t)(a.fr.id[BIN_G][u] + a.lo) : -1;
      const int64_t beg = (int64_t)(en.bl & kBegMask);
      const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
      const int64_t a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      int4 x0 = make_int4(0, 0, 0, 0), x1 = make_int4(0, 0, 0, 0);
      if (sub < nvec) x0 = ld_col4(col + a0 + 4 * sub, pol);
      if (sub + 8 < nvec) x1 = ld_col4(col + a0 + 4 * (sub + 8), pol);
      if (sub < nvec) red_group<LOOPS>(F, rep, hot_lim, copy, x0, a0 + 4 * sub, beg, end, gi, en.v, fpol);
      if (sub + 8 < nvec) red_group<LOOPS>(F, rep, hot_lim, copy, x1, a0 + 4 * (sub + 8), beg, end, gi, en.v, fpol);
    }
  }
  // ---- bin T (1..8 links): one thread per row; <= 3 int4 groups
  {
    const int64_t u1 = U[BIN_T];
    for (int64_t u = 32 * w + lane; u < u1; u += 32 * W) {
      const Entry en = a.fr.ent[BIN_T][u];
      const int32_t gi = LOOPS ? (int32_t)(a.fr.id[BIN_T][u] + a.lo) : -1;
      const int64_t beg = (int64_t)(en.bl & kBegMask);
      const int64_t end = beg + (int64_t)(en.bl >> kLenShift);
      const int64_t a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      const int4 x0 = ld_col4(col + a0, pol);
      int4 x1 = make_int4(0, 0, 0, 0), x2 = make_int4(0, 0, 0, 0);
      if (nvec > 1) x1 = ld_col4(col + a0 + 4, pol);
      if (nvec > 2) x2 = ld_col4(col + a0 + 8, pol);
      red_group<LOOPS>(F, rep, hot_lim, copy, x0, a0, beg, end, gi, en.v, fpol);
      if (nvec > 1) red_group<LOOPS>(F, rep, hot_lim, copy, x1, a0 + 4, beg, end, gi, en.v, fpol);
      if (nvec > 2) red_group<LOOPS>(F, rep, hot_lim, copy, x2, a0 + 8, beg, end, gi, en.v, fpol);
    }
  }
  // ---- every block reduces its slice of the select partials; the last block to finish
  //      finalises the sweep (DI_AUTO: k_pull, launched next, does)
  if (mode != MODE_PUSH) return;
  slice_partials(a, blockIdx.x, gridDim.x, kPushThreads);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  finalize_sweep(a, gridDim.x, kPushThreads);
}

// ------------------------------------------------------------------ pull (a5')
// F_j += sum_{i in in(j), i != j} S_i over the CSC, no atomics except for the partial sums of
// chunked hub rows. Deterministic for every row below kPullChunk in-links.
__device__ __forceinline__ double sum_group(const double *__restrict__ S, int4 x, int64_t p0,
                                            int64_t beg, int64_t end, int32_t j) {
  const int32_t ii[4] = {x.x, x.y, x.z, x.w};
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end && ii[c] != j) acc += __ldg(S + ii[c]);
  }
  return acc;
}

__global__ void __launch_bounds__(kPushThreads) k_pull(const SweepArgs a) {
  __shared__ bool s_last;
  Scalars *sc = a.sc;
  if (sc->stop) return;
  const int mode = sc->mode;
  const bool work = mode == MODE_PULL || (int64_t)sc->fill_links[0] > sc->pull_thr;
  if (work) {
    const uint64_t pol = policy_evict_first();
    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t)gridDim.x * (kPushThreads / 32);
    const int64_t w = (int64_t)blockIdx.x * (kPushThreads / 32) + (threadIdx.x >> 5);
    const int32_t *__restrict__ row = a.csc_row;
    const double *__restrict__ S = a.S;
    double *__restrict__ F = a.F;
    // ---- P3 / P2: warp per row or hub chunk
    for (int b = kPullBins - 1; b >= 2; b--) {
      const int64_t U = a.pe_count[b];
      for (int64_t u = w; u < U; u += W) {   // round-robin: rows are sorted by size
        const PullEntry en = a.pe[b][u];
        const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
        const int nvec = (int)((end - a0 + 3) >> 2);
        double acc = 0.0;
        for (int vb = 0; vb < nvec; vb += 64) {
          const int v0 = vb + lane, v1 = vb + 32 + lane;
          int4 x0 = make_int4(0, 0, 0, 0), x1 = make_int4(0, 0, 0, 0);
          if (v0 < nvec) x0 = ld_col4(row + a0 + 4 * (int64_t)v0, pol);
          if (v1 < nvec) x1 = ld_col4(row + a0 + 4 * (int64_t)v1, pol);
          if (v0 < nvec) acc += sum_group(S, x0, a0 + 4 * (int64_t)v0, beg, end, en.j);
          if (v1 < nvec) acc += sum_group(S, x1, a0 + 4 * (int64_t)v1, beg, end, en.j);
        }
        acc = warp_sum(acc);
        if (lane == 0) {
          if (b == 3)
            atomicAdd(F + en.j, acc);
          else
            F[en.j] += acc;
        }
      }
    }
    // ---- P1: 8-lane group per row (warp-uniform loop, 4 rows per step)
    {
      const int64_t U = a.pe_count[1];
      const int64_t u1 = U;
      const int sub = lane & 7;
      for (int64_t ub = 4 * w; ub < u1; ub += 4 * W) {
        const int64_t u = ub + (lane >> 3);
        double acc = 0.0;
        PullEntry en;
        en.j = -1;
        if (u < u1) {
          en = a.pe[1][u];
          const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
          const int nvec = (int)((end - a0 + 3) >> 2);
          for (int vb = sub; vb < nvec; vb += 16) {
            int4 x0 = ld_col4(row + a0 + 4 * (int64_t)vb, pol);
            int4 x1 = make_int4(0, 0, 0, 0);
            if (vb + 8 < nvec) x1 = ld_col4(row + a0 + 4 * (int64_t)(vb + 8), pol);
            acc += sum_group(S, x0, a0 + 4 * (int64_t)vb, beg, end, en.j);
            if (vb + 8 < nvec) acc += sum_group(S, x1, a0 + 4 * (int64_t)(vb + 8), beg, end, en.j);
          }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        if (sub == 0 && u < u1) F[en.j] += acc;
      }
    }
    // ---- P0: one thread per row (<= kPullT in-links, <= 3 int4 groups)
    {
      const int64_t U = a.pe_count[0];
      for (int64_t u = 32 * w + lane; u < U; u += 32 * W) {
        const PullEntry en = a.pe[0][u];
        const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
        const int nvec = (int)((end - a0 + 3) >> 2);
        const int4 x0 = ld_col4(row + a0, pol);
        int4 x1 = make_int4(0, 0, 0, 0), x2 = make_int4(0, 0, 0, 0);
        if (nvec > 1) x1 = ld_col4(row + a0 + 4, pol);
        if (nvec > 2) x2 = ld_col4(row + a0 + 8, pol);
        double acc = sum_group(S, x0, a0, beg, end, en.j);
        if (nvec > 1) acc += sum_group(S, x1, a0 + 4, beg, end, en.j);
        if (nvec > 2) acc += sum_group(S, x2, a0 + 8, beg, end, en.j);
        F[en.j] += acc;
      }
    }
  }
  // ---- slices of the select partials; the last block finalises (pull and auto modes)
  slice_partials(a, blockIdx.x, gridDim.x, kPushThreads);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  finalize_sweep(a, gridDim.x, kPushThreads);
}

template <bool LOOPS, int MINB>
void launch_push_t(const Graph &g, const SweepArgs &a) {
  static const int occ = occupancy(k_push<LOOPS, MINB>, kPushThreads);  // once, thread-safe
  k_push<LOOPS, MINB><<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a);
}

}  // namespace

int64_t select_tiles(int64_t n) { return (n + kSelTile - 1) / kSelTile; }

di_status alloc_state(Graph &g) {
  const int64_t n = g.n;
  const int64_t nt = select_tiles(n);
  DI_CK(dmalloc(&g.F, (size_t)n * 8));
  DI_CK(dmalloc(&g.H, (size_t)n * 8));
  DI_CK(dmemset(g.H, 0, (size_t)n * 8));
  DI_CK(dmemset(g.F, 0, (size_t)n * 8));
  DI_CK(dmalloc(&g.sc, sizeof(Scalars)));
  DI_CK(dmemset(g.sc, 0, sizeof(Scalars)));
  DI_CK(pinned_scalars_get(&g.sc_host));
  memset(g.sc_host, 0, sizeof(Scalars));
  DI_CK(dmalloc(&g.partials, (size_t)nt * 4 * 8));
  DI_CK(dmalloc(&g.ipartials, (size_t)nt * 4 * 8));
  DI_CK(dmalloc(&g.ppartials, (size_t)kMaxSlices * 8 * 8));
  const int rg = reduce_grid(n, g.num_sms);
  DI_CK(dmalloc(&g.red_partials, (size_t)rg * 8));
  // frontier: per-bin capacity = rows (chunks for C) whose static degree falls in the bin
  g.ntiles = nt;
  unsigned long long *cap = nullptr;
  DI_CK(dmalloc(&cap, kBins * 8));
  DI_CK(cudaMemsetAsync(cap, 0, kBins * 8, g.stream));
  k_tile_caps<<<(unsigned)nt, kSelThreads, 0, g.stream>>>(g.deg, n, cap);
  unsigned long long hcap[kBins];
  DI_CK(cudaMemcpyAsync(hcap, cap, kBins * 8, cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  dfree(cap);
  for (int b = 0; b < kBins; b++) {
    const int64_t acc = (int64_t)hcap[b];
    g.fr.cap[b] = acc;
    const size_t cap_b = (size_t)std::max<int64_t>(acc, 1);
    DI_CK(dmalloc(&g.fr.ent[b], cap_b * sizeof(Entry)));
    DI_CK(dmalloc(&g.fr.id[b], cap_b * 4));
  }
  DI_CK(dmalloc(&g.log_r, (size_t)kLogCap * 8));
  DI_CK(dmalloc(&g.log_sel, (size_t)kLogCap * 8));
  DI_CK(dmalloc(&g.log_links, (size_t)kLogCap * 8));
  DI_CK(dmalloc(&g.log_mode, (size_t)kLogCap));
  return DI_OK;
}

void launch_init(Graph &g, const double *B, double d, int64_t *launches) {
  const int64_t n = g.n;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)g.num_sms * 16);
  if (grid < 1) grid = 1;
  k_init<<<grid, 256, 0, g.stream>>>(g.F, g.H, B, (1.0 - d) / (double)g.n_global, n);
  k_reduce<<<reduce_grid(n, g.num_sms), kRedThreads, 0, g.stream>>>(g.F, n, g.red_partials, g.sc, 1);
  *launches += 2;
}

void launch_reduce_F(Graph &g, int64_t *launches) {
  k_reduce<<<reduce_grid(g.n, g.num_sms), kRedThreads, 0, g.stream>>>(g.F, g.n, g.red_partials,
                                                                     g.sc, 0);
  *launches += 1;
}

void launch_reduce_F_setr(Graph &g, int64_t *launches) {
  k_reduce<<<reduce_grid(g.n, g.num_sms), kRedThreads, 0, g.stream>>>(g.F, g.n, g.red_partials,
                                                                     g.sc, 1);
  *launches += 1;
}

void launch_select(Graph &g, int test_mode, int64_t *launches, int blk, int blocks) {
  const SweepArgs a = sweep_args(g, test_mode, blk, blocks);
  const unsigned grid = (unsigned)std::max<int64_t>(1, a.t1 - a.t0);
  if (g.has_loops)
    k_select<true><<<grid, kSelThreads, 0, g.stream>>>(a);
  else
    k_select<false><<<grid, kSelThreads, 0, g.stream>>>(a);
  *launches += 1;
}

void launch_push(Graph &g, int64_t *launches, int blk, int blocks) {
  const SweepArgs a = sweep_args(g, 0, blk, blocks);
  if (g.has_loops)
    launch_push_t<true, 4>(g, a);
  else if (g.push_occ >= 6)
    launch_push_t<false, 6>(g, a);
  else if (g.push_occ == 5)
    launch_push_t<false, 5>(g, a);
  else if (g.push_occ == 3)
    launch_push_t<false, 3>(g, a);
  else
    launch_push_t<false, 4>(g, a);
  *launches += 1;
}

void launch_pull(Graph &g, int64_t *launches) {
  const SweepArgs a = sweep_args(g, 0);
  static const int occ = occupancy(k_pull, kPushThreads);
  k_pull<<<g.num_sms * occ, kPushThreads, 0, g.stream>>>(a);
  *launches += 1;
}

// Static pull entries from the CSC (built once per graph, on the host from col_ptr).
// the pull variant's static entries per in-degree bin, built on the device: pass 0 counts the
// entries of every bin, pass 1 writes them (unordered: each entry is independent; bin P3's chunks
// are summed with fp64 atomics anyway)
__global__ void k_pull_entries(const int64_t *__restrict__ cp, int64_t n, int pass,
                               unsigned long long *__restrict__ cnt, PullEntry *e0, PullEntry *e1,
                               PullEntry *e2, PullEntry *e3) {
  const int lane = threadIdx.x & 31;
  for (int64_t j0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; j0 < n;
       j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + lane;
    int64_t beg = 0, len = 0;
    if (j < n) {
      beg = cp[j];
      len = cp[j + 1] - beg;
    }
    const int b = len == 0 ? -1 : (len <= kPullT ? 0 : (len <= kPullG ? 1 : (len <= kPullChunk ? 2 : 3)));
    const int64_t ne = b < 0 ? 0 : (b < 3 ? 1 : (len + kPullChunk - 1) / kPullChunk);
#pragma unroll
    for (int c = 0; c < kPullBins; c++) {
      const bool mine = b == c;
      // inclusive scan of the lanes' entry counts in this bin: one reservation per warp and bin
      int64_t incl = mine ? ne : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      const int64_t tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tot == 0) continue;
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(cnt + 16 * c, (unsigned long long)tot);
      base = __shfl_sync(0xffffffffu, base, 31);
      if (pass == 1 && mine) {
        PullEntry *e = c == 0 ? e0 : (c == 1 ? e1 : (c == 2 ? e2 : e3));
        int64_t at = (int64_t)base + incl - ne;
        for (int64_t k = 0; k < len; k += kPullChunk, at++)
          e[at] = PullEntry{beg + k, (int32_t)(len - k < kPullChunk ? len - k : kPullChunk), (int32_t)j};
      }
    }
  }
}

// static work entries of the rows of `ptr` (n rows) per bin, on the device
di_status build_bin_entries(Graph &g, const int64_t *ptr, int64_t n, PullEntry **out, int64_t *counts) {
  unsigned long long *cnt = nullptr;
  DI_CK(dmalloc(&cnt, kPullBins * 16 * 8));
  DI_CK(cudaMemsetAsync(cnt, 0, kPullBins * 16 * 8, g.stream));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)g.num_sms * 8));
  k_pull_entries<<<grid, 256, 0, g.stream>>>(ptr, n, 0, cnt, nullptr, nullptr, nullptr, nullptr);
  unsigned long long hc[kPullBins * 16];
  DI_CK(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  for (int b = 0; b < kPullBins; b++) {
    counts[b] = (int64_t)hc[16 * b];
    DI_CK(dmalloc(&out[b], (size_t)std::max<int64_t>(counts[b], 1) * sizeof(PullEntry)));
  }
  DI_CK(cudaMemsetAsync(cnt, 0, kPullBins * 16 * 8, g.stream));
  k_pull_entries<<<grid, 256, 0, g.stream>>>(ptr, n, 1, cnt, out[0], out[1], out[2], out[3]);
  DI_CK(cudaStreamSynchronize(g.stream));
  dfree(cnt);
  return DI_OK;
}

di_status alloc_pull(Graph &g) {
  if (!g.has_csc || g.pe[0]) return DI_OK;
  di_status s = build_bin_entries(g, g.csc_ptr, g.n, g.pe, g.pe_count);
  if (s != DI_OK) return s;
  DI_CK(dmalloc(&g.S, (size_t)std::max<int64_t>(g.n, 1) * 8));
  return DI_OK;
}

// DI_GRAPH_LOOP: condition of the device-side while node, evaluated after every cycle
__global__ void k_loop_cond(const Scalars *sc, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (sc->stop == 0 && sc->sweeps < sc->max_sweeps) ? 1u : 0u);
}

void launch_loop_cond(Graph &g, cudaGraphConditionalHandle h) {
  k_loop_cond<<<1, 1, 0, g.stream>>>(g.sc, h);
}

void launch_finalize(Graph &g, int64_t *launches) {
  const SweepArgs a = sweep_args(g, 1);
  k_finalize<<<1, kPushThreads, 0, g.stream>>>(a);
  *launches += 1;
}

}  // namespace di
