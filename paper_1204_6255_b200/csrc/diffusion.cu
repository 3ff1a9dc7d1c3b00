// diffusion.cu — the D-iteration hot path on sm_100a.
//
// One bulk-synchronous sweep n (R1) is two kernels:
//   k_select  (a2+a3+a4): for every node i, test F_i against the DI-SOP threshold
//             (r_n/L)*#out_i (literal order, reading G4) or 0 (DI-CYC);
//             for selected i: T_i = F_i, or F_i*#out_i/(#out_i - k_i*d) with k_i self-loops
//             (reading G6); H_i += T_i; F_i = 0; dangling: e += T_i
//             (P:266-267); else emit (i, v_i = T_i*d/#out_i) into the degree bin of #out_i.
//             Emission order is deterministic (ascending i inside each bin) through a
//             single-pass decoupled look-back scan over tiles. The same pass reduces
//             q = sum of unselected F and s = sum T_i*d*(#out_i-k_i)/#out_i, so that
//             r_{n+1} = q + s is known when the sweep ends (a2) without another pass over F.
//   k_push    (a5): F_j += v_i for every link i -> j, j != i, fp64 RED atomics,
//             degree-binned: CTA-chunk / warp / 8-lane group / thread per node.
// The last block of k_select finalises the sweep (deterministic fixed-order reductions,
// convergence test, starvation guard G5), so the host never has to read anything between
// sweeps: kernels of later sweeps no-op once `stop` is set.
#include "di_common.cuh"

namespace di {
namespace {

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// streaming read of the column index array: read once per sweep, do not pollute L1/L2
__device__ __forceinline__ int32_t ld_col(const int32_t *p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void red_add_f64(double *p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ int bin_of(int o) {
  return o <= kBinT ? BIN_T : (o <= kBinG ? BIN_G : (o <= kBinW ? BIN_W : BIN_C));
}

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
struct SelectArgs {
  double *F, *H;
  const int32_t *deg, *kloop;
  int64_t n;            // owned nodes
  int64_t ntiles;
  double L_total;       // global link count, as double (threshold r/L)
  double d, tol;
  int variant, paper_err, trace, test_mode;
  Scalars *sc;
  Frontier fr;
  double *partials;     // 3 per tile
  uint32_t *tflag;
  int64_t *tagg, *tincl;  // kBins per tile
  double *log_r;
  int64_t *log_sel, *log_links;
  uint8_t *log_mode;
};

// Decoupled look-back (single-pass scan): warp 0 of tile `tile` obtains the exclusive
// prefix of the 4 bin counts. Flags are tagged with the select-launch epoch so they never
// need resetting: flag = epoch << 2 | {1: aggregate ready, 2: inclusive prefix ready}.
__device__ __forceinline__ void lookback(const SelectArgs &a, int64_t tile, uint32_t epoch,
                                         const int64_t agg[kBins], int64_t excl[kBins]) {
  const int lane = threadIdx.x & 31;
  const uint32_t tag = epoch << 2;
  if (tile == 0) {
    if (lane < kBins) a.tincl[lane] = agg[lane];
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_u32(a.tflag, tag | 2u);
#pragma unroll
    for (int b = 0; b < kBins; b++) excl[b] = 0;
    return;
  }
  if (lane < kBins) a.tagg[tile * kBins + lane] = agg[lane];
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release_u32(a.tflag + tile, tag | 1u);
  int64_t run[kBins] = {0, 0, 0, 0};
  int64_t pred = tile - 1;
  while (true) {
    const int64_t idx = pred - lane;
    uint32_t f = tag | 2u;
    if (idx >= 0) {
      do {
        f = ld_acquire_u32(a.tflag + idx);
      } while ((f & ~3u) != tag || (f & 3u) == 0);
    }
    const bool isP = (f & 3u) == 2u;
    const uint32_t pm = __ballot_sync(0xffffffffu, isP);
    const int stop_lane = pm ? (__ffs(pm) - 1) : 32;
    int64_t v[kBins] = {0, 0, 0, 0};
    if (idx >= 0 && lane <= stop_lane) {
      const int64_t *src = (lane == stop_lane) ? (a.tincl + idx * kBins) : (a.tagg + idx * kBins);
#pragma unroll
      for (int b = 0; b < kBins; b++) v[b] = __ldcg(src + b);
    }
#pragma unroll
    for (int b = 0; b < kBins; b++) run[b] += warp_sum(v[b]);
    if (pm) break;
    pred -= 32;
  }
  if (lane < kBins) {
    int64_t mine = 0;
#pragma unroll
    for (int b = 0; b < kBins; b++)
      if (b == lane) mine = run[b] + agg[b];
    a.tincl[tile * kBins + lane] = mine;
  }
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release_u32(a.tflag + tile, tag | 2u);
#pragma unroll
  for (int b = 0; b < kBins; b++) excl[b] = run[b];
}

template <bool LOOPS>
__global__ void __launch_bounds__(kSelThreads) k_select(const SelectArgs a) {
  constexpr int NW = kSelThreads / 32;
  __shared__ uint32_t s_tile;
  __shared__ int s_wcnt[NW][kBins];
  __shared__ int64_t s_excl[kBins];
  __shared__ double s_red[NW][3];
  __shared__ int64_t s_links[NW];
  __shared__ int s_sel[NW], s_selnd[NW];
  __shared__ bool s_last;

  Scalars *sc = a.sc;
  if (!a.test_mode && sc->stop) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->active = 0;
    return;
  }
  const uint32_t epoch = sc->epoch;
  const int par = epoch & 1;
  if (threadIdx.x == 0) s_tile = atomicAdd(&sc->tile_ctr[par], 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double r = sc->r;
  const bool cyc = (a.variant == DI_CYC) || sc->guard;
  const double d = a.d;
  const double t = (a.L_total > 0.0) ? r / a.L_total : 0.0;  // r/L once (G3, G4)
  const int64_t base = tile * (int64_t)kSelTile + (int64_t)threadIdx.x * kSelItems;

  double f[kSelItems];
  int o[kSelItems];
  int kl[kSelItems];
  if (base + kSelItems <= a.n) {
    const double2 *F2 = reinterpret_cast<const double2 *>(a.F + base);
#pragma unroll
    for (int j = 0; j < kSelItems / 2; j++) {
      double2 x = F2[j];
      f[2 * j] = x.x;
      f[2 * j + 1] = x.y;
    }
    const int4 *D4 = reinterpret_cast<const int4 *>(a.deg + base);
#pragma unroll
    for (int j = 0; j < kSelItems / 4; j++) {
      int4 x = D4[j];
      o[4 * j] = x.x;
      o[4 * j + 1] = x.y;
      o[4 * j + 2] = x.z;
      o[4 * j + 3] = x.w;
    }
    if (LOOPS) {
      const int4 *K4 = reinterpret_cast<const int4 *>(a.kloop + base);
#pragma unroll
      for (int j = 0; j < kSelItems / 4; j++) {
        int4 x = K4[j];
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
      o[j] = (i < a.n) ? a.deg[i] : 0;
      if (LOOPS) kl[j] = (i < a.n) ? a.kloop[i] : 0;
    }
  }
  if (!LOOPS) {
#pragma unroll
    for (int j = 0; j < kSelItems; j++) kl[j] = 0;
  }

  double v[kSelItems];
  uint32_t selmask = 0;
  int cnt[kBins] = {0, 0, 0, 0};
  double q = 0.0, s = 0.0, e = 0.0;
  int64_t links = 0;
  int nsel = 0, nsel_nd = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; j++) {
    const int64_t i = base + j;
    v[j] = 0.0;
    if (i >= a.n) continue;
    const double od = (double)o[j];
    const double thr = cyc ? 0.0 : __dmul_rn(t, od);  // (r/L)*out[i]
    if (f[j] > thr) {                                   // strict '>'
      double T = f[j];
      if (LOOPS && kl[j] > 0)                           // P:259-263 with k copies (G6)
        T = __ddiv_rn(__dmul_rn(f[j], od), __dsub_rn(od, __dmul_rn((double)kl[j], d)));
      a.H[i] = __dadd_rn(a.H[i], T);
      a.F[i] = 0.0;
      nsel++;
      if (o[j] == 0) {
        e = __dadd_rn(e, T);
      } else {
        const double Td = __dmul_rn(T, d);
        v[j] = __ddiv_rn(Td, od);                       // sent = transit*d/out[i]
        s = __dadd_rn(s, __ddiv_rn(__dmul_rn(Td, (double)(o[j] - kl[j])), od));
        links += o[j];
        nsel_nd++;
        const int b = bin_of(o[j]);
        cnt[b] += (b == BIN_C) ? (o[j] + kChunk - 1) / kChunk : 1;
        selmask |= 1u << j;
      }
    } else {
      q = __dadd_rn(q, f[j]);
    }
  }

  // ---- block-wide exclusive scan of the 4 bin counts
  int incl[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) {
    int x = cnt[b];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    incl[b] = x;
    if (lane == 31) s_wcnt[warp][b] = x;
  }
  // ---- block reductions of q, s, e, links, selected (fixed order)
  q = warp_sum(q);
  s = warp_sum(s);
  e = warp_sum(e);
  links = warp_sum(links);
  nsel = warp_sum(nsel);
  nsel_nd = warp_sum(nsel_nd);
  if (lane == 0) {
    s_red[warp][0] = q;
    s_red[warp][1] = s;
    s_red[warp][2] = e;
    s_links[warp] = links;
    s_sel[warp] = nsel;
    s_selnd[warp] = nsel_nd;
  }
  __syncthreads();
  int texcl[kBins];
  int64_t agg[kBins];
#pragma unroll
  for (int b = 0; b < kBins; b++) {
    int we = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NW; w++) {
      const int c = s_wcnt[w][b];
      we += (w < warp) ? c : 0;
      tot += c;
    }
    texcl[b] = we + incl[b] - cnt[b];
    agg[b] = tot;
  }
  if (warp == 0) {
    int64_t ex[kBins];
    lookback(a, tile, epoch, agg, ex);
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < kBins; b++) s_excl[b] = ex[b];
      if (tile == a.ntiles - 1) {
#pragma unroll
        for (int b = 0; b < kBins; b++) sc->bin_count[b] = ex[b] + agg[b];
      }
    }
  }
  if (threadIdx.x == 32) {
    double tq = 0.0, ts = 0.0, te = 0.0;
    int64_t tl = 0;
    int tsel = 0, tnd = 0;
    for (int w = 0; w < NW; w++) {
      tq += s_red[w][0];
      ts += s_red[w][1];
      te += s_red[w][2];
      tl += s_links[w];
      tsel += s_sel[w];
      tnd += s_selnd[w];
    }
    a.partials[tile * 3 + 0] = tq;
    a.partials[tile * 3 + 1] = ts;
    a.partials[tile * 3 + 2] = te;
    if (tl) atomicAdd((unsigned long long *)&sc->sweep_links, (unsigned long long)tl);
    if (tsel) atomicAdd((unsigned long long *)&sc->sweep_sel, (unsigned long long)tsel);
    if (tnd) atomicAdd((unsigned long long *)&sc->sweep_sel_nd, (unsigned long long)tnd);
  }
  __syncthreads();

  // ---- emit (i, v_i) in ascending i inside each bin
  if (selmask) {
    int64_t pos[kBins];
#pragma unroll
    for (int b = 0; b < kBins; b++) pos[b] = s_excl[b] + texcl[b];
#pragma unroll
    for (int j = 0; j < kSelItems; j++) {
      if (!(selmask & (1u << j))) continue;
      const int32_t i = (int32_t)(base + j);
      const int b = bin_of(o[j]);
      if (b != BIN_C) {
        a.fr.ids[b][pos[b]] = i;
        a.fr.val[b][pos[b]] = v[j];
        pos[b]++;
      } else {
        const int nch = (o[j] + kChunk - 1) / kChunk;
        for (int c = 0; c < nch; c++) {
          a.fr.ids[BIN_C][pos[BIN_C] + c] = i;
          a.fr.val[BIN_C][pos[BIN_C] + c] = v[j];
          a.fr.chunk[pos[BIN_C] + c] = c;
        }
        pos[BIN_C] += nch;
      }
    }
  }

  // ---- last block finalises the sweep
  __threadfence();
  if (threadIdx.x == 0) s_last = atomicAdd(&sc->ticket, 1u) == (uint32_t)(a.ntiles - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double aq = 0.0, as = 0.0, ae = 0.0;
  for (int64_t tt = threadIdx.x; tt < a.ntiles; tt += kSelThreads) {
    aq += __ldcg(a.partials + tt * 3 + 0);
    as += __ldcg(a.partials + tt * 3 + 1);
    ae += __ldcg(a.partials + tt * 3 + 2);
  }
  aq = warp_sum(aq);
  as = warp_sum(as);
  ae = warp_sum(ae);
  if (lane == 0) {
    s_red[warp][0] = aq;
    s_red[warp][1] = as;
    s_red[warp][2] = ae;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tq = 0.0, ts = 0.0, te = 0.0;
    for (int w = 0; w < NW; w++) {
      tq += s_red[w][0];
      ts += s_red[w][1];
      te += s_red[w][2];
    }
    volatile Scalars *vs = sc;
    const int64_t sel = vs->sweep_sel, lk = vs->sweep_links, nd = vs->sweep_sel_nd;
    const int64_t sw = vs->sweeps;
    if (a.trace && sw < kLogCap) {
      a.log_r[sw] = r;
      a.log_sel[sw] = sel;
      a.log_links[sw] = lk;
      a.log_mode[sw] = 0;
    }
    const double r_next = tq + ts;   // r_{n+1} = q_n + s_n (a2)
    const double e_tot = vs->e + te;
    vs->e = e_tot;
    vs->q = tq;
    vs->s = ts;
    vs->e_sw = te;
    vs->r = r_next;
    vs->sweeps = sw + 1;
    vs->selected_total = vs->selected_total + sel;
    vs->selected_nd_total = vs->selected_nd_total + nd;
    vs->links_total = vs->links_total + lk;
    vs->scanned_total = vs->scanned_total + a.n;
    if (cyc && a.variant != DI_CYC) vs->guards = vs->guards + 1;
    const double err = a.paper_err ? r_next / (1.0 - d - d * e_tot) : r_next;
    const int stop = err <= a.tol;
    vs->stop = stop;
    vs->guard = (sel == 0 && !stop && a.variant == DI_SOP) ? 1 : 0;
    int64_t tot = 0;
    for (int b = 0; b < kBins; b++) tot += vs->bin_count[b];
    vs->active = tot > 0;
    vs->sweep_sel = 0;
    vs->sweep_links = 0;
    vs->sweep_sel_nd = 0;
    vs->tile_ctr[par ^ 1] = 0;
    vs->ticket = 0;
    vs->epoch = epoch + 1;
  }
}

// ------------------------------------------------------------------ push (a5)
struct PushArgs {
  Frontier fr;
  const int64_t *row_ptr;
  const int32_t *col;
  double *F;
  int64_t lo;  // global id of local node 0 (self-loop test compares global ids)
  Scalars *sc;
};

// one warp walks links [beg, end) of node gi, adding v to each target
__device__ __forceinline__ void warp_row(const int32_t *__restrict__ col, double *__restrict__ F,
                                         int64_t beg, int64_t end, int32_t gi, double v, int lane,
                                         uint64_t pol) {
  int64_t k = beg + lane;
  for (; k + 96 < end; k += 128) {
    const int32_t j0 = ld_col(col + k, pol), j1 = ld_col(col + k + 32, pol);
    const int32_t j2 = ld_col(col + k + 64, pol), j3 = ld_col(col + k + 96, pol);
    if (j0 != gi) red_add_f64(F + j0, v);
    if (j1 != gi) red_add_f64(F + j1, v);
    if (j2 != gi) red_add_f64(F + j2, v);
    if (j3 != gi) red_add_f64(F + j3, v);
  }
  for (; k < end; k += 32) {
    const int32_t j = ld_col(col + k, pol);
    if (j != gi) red_add_f64(F + j, v);
  }
}

__global__ void __launch_bounds__(kPushThreads) k_push(const PushArgs a) {
  Scalars *sc = a.sc;
  if (!sc->active) return;
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kPushThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kPushThreads / 32) + (threadIdx.x >> 5);
  const int64_t *__restrict__ rp = a.row_ptr;
  double *__restrict__ F = a.F;
  // ---- bin C: hub rows, fixed-size chunks of kChunk links, one warp per chunk
  {
    const int64_t U = sc->bin_count[BIN_C];
    const int64_t u0 = w * U / W, u1 = (w + 1) * U / W;
    for (int64_t u = u0; u < u1; u++) {
      const int32_t i = a.fr.ids[BIN_C][u];
      const double v = a.fr.val[BIN_C][u];
      const int64_t beg = rp[i] + (int64_t)a.fr.chunk[u] * kChunk;
      const int64_t end = min(beg + (int64_t)kChunk, rp[i + 1]);
      warp_row(a.col, F, beg, end, (int32_t)(i + a.lo), v, lane, pol);
    }
  }
  // ---- bin W: one warp per node
  {
    const int64_t U = sc->bin_count[BIN_W];
    const int64_t u0 = w * U / W, u1 = (w + 1) * U / W;
    for (int64_t u = u0; u < u1; u++) {
      const int32_t i = a.fr.ids[BIN_W][u];
      const double v = a.fr.val[BIN_W][u];
      warp_row(a.col, F, rp[i], rp[i + 1], (int32_t)(i + a.lo), v, lane, pol);
    }
  }
  // ---- bin G: 8-lane group per node, 4 nodes per warp step
  {
    const int64_t U = sc->bin_count[BIN_G];
    const int64_t u0 = w * U / W, u1 = (w + 1) * U / W;
    const int sub = lane & 7;
    for (int64_t u = u0 + (lane >> 3); u < u1; u += 4) {
      const int32_t i = a.fr.ids[BIN_G][u];
      const double v = a.fr.val[BIN_G][u];
      const int32_t gi = (int32_t)(i + a.lo);
      const int64_t end = rp[i + 1];
      for (int64_t k = rp[i] + sub; k < end; k += 8) {
        const int32_t j = ld_col(a.col + k, pol);
        if (j != gi) red_add_f64(F + j, v);
      }
    }
  }
  // ---- bin T: one thread per node
  {
    const int64_t U = sc->bin_count[BIN_T];
    const int64_t u0 = w * U / W, u1 = (w + 1) * U / W;
    for (int64_t u = u0 + lane; u < u1; u += 32) {
      const int32_t i = a.fr.ids[BIN_T][u];
      const double v = a.fr.val[BIN_T][u];
      const int32_t gi = (int32_t)(i + a.lo);
      const int64_t beg = rp[i], end = rp[i + 1];
      int32_t js[kBinT];
#pragma unroll
      for (int k = 0; k < kBinT; k++) js[k] = (beg + k < end) ? ld_col(a.col + beg + k, pol) : gi;
#pragma unroll
      for (int k = 0; k < kBinT; k++)
        if (js[k] != gi) red_add_f64(F + js[k], v);
    }
  }
}

int push_grid(const Graph &g) {
  static int occ = 0;
  if (occ == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_push, kPushThreads, 0);
    if (occ < 1) occ = 1;
  }
  return g.num_sms * occ;
}

}  // namespace

int64_t select_tiles(int64_t n) { return (n + kSelTile - 1) / kSelTile; }

di_status alloc_state(Graph &g) {
  const int64_t n = g.n;
  const int64_t nt = select_tiles(n);
  DI_CK(cudaMalloc(&g.F, (size_t)n * 8));
  DI_CK(cudaMalloc(&g.H, (size_t)n * 8));
  DI_CK(cudaMemset(g.H, 0, (size_t)n * 8));
  DI_CK(cudaMemset(g.F, 0, (size_t)n * 8));
  DI_CK(cudaMalloc(&g.sc, sizeof(Scalars)));
  DI_CK(cudaMemset(g.sc, 0, sizeof(Scalars)));
  DI_CK(cudaMallocHost(&g.sc_host, sizeof(Scalars)));
  memset(g.sc_host, 0, sizeof(Scalars));
  g.sc_host->epoch = 1;
  DI_CK(cudaMemcpy(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice));
  DI_CK(cudaMalloc(&g.partials, (size_t)nt * 3 * 8));
  const int rg = reduce_grid(n, g.num_sms);
  DI_CK(cudaMalloc(&g.red_partials, (size_t)rg * 8));
  DI_CK(cudaMalloc(&g.tile_flag, (size_t)nt * 4));
  DI_CK(cudaMemset(g.tile_flag, 0, (size_t)nt * 4));
  DI_CK(cudaMalloc(&g.tile_agg, (size_t)nt * kBins * 8));
  DI_CK(cudaMalloc(&g.tile_incl, (size_t)nt * kBins * 8));
  for (int b = 0; b < kBins; b++) {
    int64_t cap = n;
    if (b == BIN_C) cap = n + g.l / kChunk + 1;
    if (cap < 1) cap = 1;
    g.fr.cap[b] = cap;
    DI_CK(cudaMalloc(&g.fr.ids[b], (size_t)cap * 4));
    DI_CK(cudaMalloc(&g.fr.val[b], (size_t)cap * 8));
  }
  DI_CK(cudaMalloc(&g.fr.chunk, (size_t)g.fr.cap[BIN_C] * 4));
  DI_CK(cudaMalloc(&g.log_r, (size_t)kLogCap * 8));
  DI_CK(cudaMalloc(&g.log_sel, (size_t)kLogCap * 8));
  DI_CK(cudaMalloc(&g.log_links, (size_t)kLogCap * 8));
  DI_CK(cudaMalloc(&g.log_mode, (size_t)kLogCap));
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

void launch_select(Graph &g, double d, double tol, int variant, int paper_err, int trace,
                   int test_mode, int64_t *launches) {
  SelectArgs a;
  a.F = g.F;
  a.H = g.H;
  a.deg = g.deg;
  a.kloop = g.kloop;
  a.n = g.n;
  a.ntiles = select_tiles(g.n);
  a.L_total = (double)g.l_global;
  a.d = d;
  a.tol = tol;
  a.variant = variant;
  a.paper_err = paper_err;
  a.trace = trace;
  a.test_mode = test_mode;
  a.sc = g.sc;
  a.fr = g.fr;
  a.partials = g.partials;
  a.tflag = g.tile_flag;
  a.tagg = g.tile_agg;
  a.tincl = g.tile_incl;
  a.log_r = g.log_r;
  a.log_sel = g.log_sel;
  a.log_links = g.log_links;
  a.log_mode = g.log_mode;
  if (g.has_loops)
    k_select<true><<<(unsigned)a.ntiles, kSelThreads, 0, g.stream>>>(a);
  else
    k_select<false><<<(unsigned)a.ntiles, kSelThreads, 0, g.stream>>>(a);
  *launches += 1;
}

void launch_push(Graph &g, int64_t *launches) {
  PushArgs a;
  a.fr = g.fr;
  a.row_ptr = g.row_ptr;
  a.col = g.col;
  a.F = g.F;
  a.lo = g.lo;
  a.sc = g.sc;
  k_push<<<push_grid(g), kPushThreads, 0, g.stream>>>(a);
  *launches += 1;
}

}  // namespace di
