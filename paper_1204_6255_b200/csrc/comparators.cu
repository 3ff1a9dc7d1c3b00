// comparators.cu — the paper's comparison schemes on the GPU.
//
//   DI_PI_PULL  (PI, P:152-182 [§2.5.1]): x_new_i = (1-d)/N + sum_{j in l_in[i]} d*x_old_j/out_j,
//               pulled over the CSC (deterministic except chunked in-hubs);
//   DI_PI_PUSH  (PI', P:184-214 [§2.5.2]): the same iterate by scatter over the CSR, fp64 REDs;
//   both then: error = sum x_new; x_new += (1-error)/N;
//              error = sum |x_new - x_old| * d/(1-d); stop at error <= tol (G10:
//              PI' uses PI's rule); x_old <- x_new (G20).
//   DI_GS_BLOCK (GS, P:216-247 [§2.5.3], reading R4): kGsBlocks ordered node blocks per sweep;
//               inside a block the rows are updated from the values of the previous block
//               state (Jacobi), across blocks in order (Gauss-Seidel):
//               x_i = ((1-d)/N + sum_{j in l_in[i], j != i} d*x_j/out_j) / diag_i,
//               diag_i = 1 - k_i*(d/out_i) (self entries); error = sum(x - prev),
//               e = sum_{out=0} x, error *= d/(1-d-d*e) (G11).
// Every sweep reads all L links (the comparators' cost model). di_history returns x
// (PI/PI': normalised; GS: raw) in the caller's numbering.
#include <cmath>
#include <string>
#include <vector>

#include "di_common.cuh"
#include "kern_util.cuh"
#include "sweep.cuh"

namespace di {
namespace {

constexpr int kCmpThreads = 256;
constexpr int kGsBlocks = 32;

struct CmpArgs {
  const int32_t *deg, *kloop, *csc_row, *col;
  const int64_t *csc_ptr;
  int64_t n;
  double d, b;  // b = (1-d)/N
  Scalars *sc;
  double *partials;
  PullEntry *pe[kPullBins];
  int64_t pe_count[kPullBins];
  PullEntry *re[kPullBins];  // static out-row entries for PI' (j = source row id)
  int64_t re_count[kPullBins];
  double *rep;               // replicated accumulators of the hot ids j < hot_lim (PI' push)
  int32_t hot_lim;
};

// PI' scatter of t into xn[j]: a hot id (j < hot_lim) goes to copy `copy` of its replicated
// accumulator (same-address REDs serialise in one L2 slice), folded by k_pi_fold
__device__ __forceinline__ void pi_add(const CmpArgs &a, double *__restrict__ xn, int32_t j,
                                       double t, int copy, uint64_t fpol) {
  if (j < a.hot_lim)
    red_add_f64(a.rep + (int64_t)(copy * kHotRanks + j) * kRepStride, t);
  else
    red_add_f64_hint(xn + j, t, fpol);
}

__global__ void k_pi_fold(const CmpArgs a, double *__restrict__ xn) {
  for (int k = threadIdx.x; k < a.hot_lim; k += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < kRepCopies; c++) {
      double *p = a.rep + (int64_t)(c * kHotRanks + k) * kRepStride;
      acc += *p;
      *p = 0.0;
    }
    if (acc != 0.0) xn[k] += acc;
  }
}

// y_i = d*x_i/out_i (0 for dangling: l_out is empty), xn_i = (1-d)/N
__global__ void k_pi_prep(const CmpArgs a, const double *__restrict__ x, double *__restrict__ y,
                          double *__restrict__ xn) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int o = a.deg[i];
    y[i] = o ? a.d * x[i] / (double)o : 0.0;
    if (xn) xn[i] = a.b;
  }
}

__device__ __forceinline__ double sum_all(const double *__restrict__ y, int4 v, int64_t p0,
                                          int64_t beg, int64_t end) {
  const int32_t ii[4] = {v.x, v.y, v.z, v.w};
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 4; c++) {
    const int64_t p = p0 + c;
    if (p >= beg && p < end) acc += __ldg(y + ii[c]);
  }
  return acc;
}

// x_new_j += sum_{i in in(j)} y_i over the static pull entries (self entries included: PI)
__global__ void __launch_bounds__(kCmpThreads) k_pi_pull(const CmpArgs a, const double *__restrict__ y,
                                                         double *__restrict__ xn) {
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kCmpThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kCmpThreads / 32) + (threadIdx.x >> 5);
  for (int b = kPullBins - 1; b >= 2; b--) {
    for (int64_t u = w; u < a.pe_count[b]; u += W) {
      const PullEntry en = a.pe[b][u];
      const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      double acc = 0.0;
      for (int v = lane; v < nvec; v += 32)
        acc += sum_all(y, ld_col4(a.csc_row + a0 + 4 * (int64_t)v, pol), a0 + 4 * (int64_t)v, beg, end);
      acc = warp_sum(acc);
      if (lane == 0) {
        if (b == 3)
          atomicAdd(xn + en.j, acc);
        else
          xn[en.j] += acc;
      }
    }
  }
  for (int b = 0; b < 2; b++) {
    for (int64_t u = 32 * w + lane; u < a.pe_count[b]; u += 32 * W) {
      const PullEntry en = a.pe[b][u];
      const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      double acc = 0.0;
      for (int v = 0; v < nvec; v++)
        acc += sum_all(y, ld_col4(a.csc_row + a0 + 4 * (int64_t)v, pol), a0 + 4 * (int64_t)v, beg, end);
      xn[en.j] += acc;
    }
  }
}

// PI': x_new_j += transit_i for every link i -> j, self entries included
__global__ void __launch_bounds__(kCmpThreads) k_pi_push(const CmpArgs a, const double *__restrict__ y,
                                                         double *__restrict__ xn) {
  const uint64_t pol = policy_evict_first(), fpol = policy_evict_last();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kCmpThreads / 32);
  const int64_t w = (int64_t)blockIdx.x * (kCmpThreads / 32) + (threadIdx.x >> 5);
  const int copy = (int)(w % kRepCopies);
  for (int b = kPullBins - 1; b >= 2; b--) {
    for (int64_t u = w; u < a.re_count[b]; u += W) {
      const PullEntry en = a.re[b][u];
      const double t = y[en.j];
      if (t == 0.0) continue;
      const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      for (int v = lane; v < nvec; v += 32) {
        const int4 x = ld_col4(a.col + a0 + 4 * (int64_t)v, pol);
        const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const int64_t p = a0 + 4 * (int64_t)v + c;
          if (p >= beg && p < end) pi_add(a, xn, jj[c], t, copy, fpol);
        }
      }
    }
  }
  for (int b = 0; b < 2; b++) {
    for (int64_t u = 32 * w + lane; u < a.re_count[b]; u += 32 * W) {
      const PullEntry en = a.re[b][u];
      const double t = y[en.j];
      const int64_t beg = en.beg, end = en.beg + en.len, a0 = beg & ~3ll;
      const int nvec = (int)((end - a0 + 3) >> 2);
      for (int v = 0; v < nvec; v++) {
        const int4 x = ld_col4(a.col + a0 + 4 * (int64_t)v, pol);
        const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const int64_t p = a0 + 4 * (int64_t)v + c;
          if (p >= beg && p < end) pi_add(a, xn, jj[c], t, copy, fpol);
        }
      }
    }
  }
}

// deterministic block partials + last-block total of f(i); the total goes to *out
template <typename Fn>
__device__ void reduce_to(const CmpArgs &a, Fn f, double *out) {
  __shared__ double s_w[kCmpThreads / 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += f(i);
  acc = warp_sum(acc);
  if (lane == 0) s_w[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kCmpThreads / 32; k++) t += s_w[k];
    a.partials[blockIdx.x] = t;
    __threadfence();
    s_last = atomicAdd(&a.sc->red_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  acc = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += kCmpThreads) acc += __ldcg(a.partials + k);
  acc = warp_sum(acc);
  __syncthreads();
  if (lane == 0) s_w[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kCmpThreads / 32; k++) t += s_w[k];
    *out = t;
    a.sc->red_ticket = 0;
  }
}

__global__ void __launch_bounds__(kCmpThreads) k_sum(const CmpArgs a, const double *__restrict__ x,
                                                     double *out) {
  reduce_to(a, [&](int64_t i) { return x[i]; }, out);
}

// x_new_i += (1 - sum)/N; error partials |x_new - x_old|
__global__ void __launch_bounds__(kCmpThreads) k_pi_fix(const CmpArgs a, double *__restrict__ xn,
                                                        const double *__restrict__ x) {
  const double c = (1.0 - a.sc->resid) / (double)a.n;
  reduce_to(a, [&](int64_t i) {
    const double v = xn[i] + c;
    xn[i] = v;
    return fabs(v - x[i]);
  }, &a.sc->q);
}

// GS block: tmp_i for rows i in [lo, hi), warp per row over the in-links (j != i)
__global__ void __launch_bounds__(kCmpThreads) k_gs_rows(const CmpArgs a, const double *__restrict__ y,
                                                         double *__restrict__ tmp, int64_t lo,
                                                         int64_t hi) {
  const uint64_t pol = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * (kCmpThreads / 32);
  for (int64_t i = lo + (int64_t)blockIdx.x * (kCmpThreads / 32) + (threadIdx.x >> 5); i < hi; i += W) {
    const int64_t beg = a.csc_ptr[i], end = a.csc_ptr[i + 1], a0 = beg & ~3ll;
    const int nvec = (int)((end - a0 + 3) >> 2);
    double acc = 0.0;
    for (int v = lane; v < nvec; v += 32) {
      const int4 x = ld_col4(a.csc_row + a0 + 4 * (int64_t)v, pol);
      const int32_t jj[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const int64_t p = a0 + 4 * (int64_t)v + c;
        if (p >= beg && p < end && jj[c] != (int32_t)i) acc += __ldg(y + jj[c]);
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      double diag = 1.0;
      const int k = a.kloop[i], o = a.deg[i];
      for (int s = 0; s < k; s++) diag -= a.d / (double)o;     // P:233-235, once per self entry
      tmp[i] = (a.b + acc) / diag;
    }
  }
}

// GS block commit: x_i <- tmp_i, y_i = d*x_i/out_i; partials of (x_i - previous)
__global__ void __launch_bounds__(kCmpThreads) k_gs_commit(const CmpArgs a, double *__restrict__ x,
                                                           double *__restrict__ y,
                                                           const double *__restrict__ tmp,
                                                           int64_t lo, int64_t hi, double *acc_out) {
  CmpArgs b = a;
  b.n = hi - lo;
  reduce_to(b, [&](int64_t k) {
    const int64_t i = lo + k;
    const double prev = x[i], v = tmp[i];
    x[i] = v;
    const int o = a.deg[i];
    y[i] = o ? a.d * v / (double)o : 0.0;
    return v - prev;
  }, acc_out);
}

__global__ void __launch_bounds__(kCmpThreads) k_gs_dangling(const CmpArgs a, const double *__restrict__ x) {
  reduce_to(a, [&](int64_t i) { return a.deg[i] == 0 ? x[i] : 0.0; }, &a.sc->e);
}

__global__ void k_fill(double *x, double v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

di_status fail_cmp(const std::string &msg) {
  set_error(msg);
  return DI_ECUDA;
}

}  // namespace

di_status run_comparator(Graph &g, double d, double tol, int variant, int64_t max_sweeps,
                         uint32_t flags, di_stats *st) {
  (void)flags;
  if (!g.has_csc && variant != DI_PI_PUSH)
    return set_error("di_solve: PI / GS comparators need the CSC (DI_BUILD_CSC)"), DI_EINVAL;
  const int64_t n = g.n;
  const int grid = g.num_sms * 4;
  // lazily built static out-row entries (PI') and work buffers
  if (variant == DI_PI_PUSH && !g.re[0]) {   // (the same size bins as the pull's, over the CSR)
    di_status bs = build_bin_entries(g, g.row_ptr, n, g.re, g.re_count);
    if (bs != DI_OK) return bs;
  }
  if (!g.aux) DI_CK(dmalloc(&g.aux, (size_t)n * 8));
  if (!g.S) DI_CK(dmalloc(&g.S, (size_t)n * 8));
  if (!g.cmp_partials) DI_CK(dmalloc(&g.cmp_partials, (size_t)grid * 8));
  CmpArgs a;
  a.deg = g.deg;
  a.kloop = g.kloop;
  a.csc_row = g.csc_row;
  a.csc_ptr = g.csc_ptr;
  a.col = g.col;
  a.n = n;
  a.d = d;
  a.b = (1.0 - d) / (double)g.n_global;
  a.sc = g.sc;
  a.partials = g.cmp_partials;
  {  // the replicated hot accumulators of the push schedules (prepare_cycle), when present
    const SweepArgs sa = sweep_args(g, 0);
    a.rep = sa.rep;
    a.hot_lim = sa.hot_shift > 0 ? sa.hot_shift : 0;
  }
  for (int b = 0; b < kPullBins; b++) {
    a.pe[b] = g.pe[b];
    a.pe_count[b] = g.pe_count[b];
    a.re[b] = g.re[b];
    a.re_count[b] = g.re_count[b];
  }
  memset(g.sc_host, 0, sizeof(Scalars));
  DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  cudaEvent_t t0, t1;
  DI_CK(cudaEventCreate(&t0));
  DI_CK(cudaEventCreate(&t1));
  DI_CK(cudaEventRecord(t0, g.stream));
  int64_t launches = 0, iters = 0;
  double err = INFINITY;
  double *x = g.H, *xn = g.aux, *y = g.S;
  const cudaStream_t s = g.stream;
  if (variant == DI_PI_PULL || variant == DI_PI_PUSH) {
    k_fill<<<grid, 256, 0, s>>>(x, 1.0 / (double)g.n_global, n);   // x_old = 1/N
    launches++;
    while (err > tol && iters < max_sweeps) {
      k_pi_prep<<<grid, 256, 0, s>>>(a, x, y, xn);
      if (variant == DI_PI_PULL) {
        k_pi_pull<<<grid, kCmpThreads, 0, s>>>(a, y, xn);
      } else {
        k_pi_push<<<grid, kCmpThreads, 0, s>>>(a, y, xn);
        if (a.hot_lim > 0) {  // the hot ids' replicated accumulators into xn
          k_pi_fold<<<1, 256, 0, s>>>(a, xn);
          launches++;
        }
      }
      k_sum<<<grid, kCmpThreads, 0, s>>>(a, xn, &g.sc->resid);
      k_pi_fix<<<grid, kCmpThreads, 0, s>>>(a, xn, x);
      launches += 4;
      DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
      DI_CK(cudaStreamSynchronize(s));
      err = g.sc_host->q * d / (1.0 - d);
      std::swap(x, xn);                                                 // G20
      iters++;
    }
  } else {  // DI_GS_BLOCK
    k_fill<<<grid, 256, 0, s>>>(x, a.b, n);                             // x = (1-d)/N
    k_pi_prep<<<grid, 256, 0, s>>>(a, x, y, nullptr);
    launches += 2;
    std::vector<double> part(kGsBlocks);
    double *dacc = nullptr;
    DI_CK(dmalloc(&dacc, kGsBlocks * 8));
    DI_CK(cudaMemsetAsync(dacc, 0, kGsBlocks * 8, s));
    // one sweep (kGsBlocks x (rows, commit) + the dangling sum) as a CUDA graph, captured once per
    // call on a private stream and launched once per sweep: 2 kGsBlocks + 1 kernels whose launch
    // gaps dominated the sweep on small graphs (C2: 40.9 ms for GS vs 3.4 ms for DI-SOP in r1)
    cudaGraph_t sweep_g = nullptr;
    cudaGraphExec_t sweep_x = nullptr;
    int64_t per_sweep = 1;
    {
      cudaStream_t cs = nullptr;
      DI_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      DI_CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < kGsBlocks; k++) {
        const int64_t lo = n * k / kGsBlocks, hi = n * (k + 1) / kGsBlocks;
        if (lo == hi) continue;   // its partial stays 0
        k_gs_rows<<<grid, kCmpThreads, 0, cs>>>(a, y, xn, lo, hi);
        k_gs_commit<<<grid, kCmpThreads, 0, cs>>>(a, x, y, xn, lo, hi, dacc + k);
        per_sweep += 2;
      }
      k_gs_dangling<<<grid, kCmpThreads, 0, cs>>>(a, x);
      cudaError_t ce = cudaStreamEndCapture(cs, &sweep_g);
      cudaStreamDestroy(cs);
      if (ce != cudaSuccess) return fail_cmp(std::string("GS sweep capture: ") + cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&sweep_x, sweep_g, 0);
      if (ce != cudaSuccess) {
        cudaGraphDestroy(sweep_g);
        return fail_cmp(std::string("GS sweep instantiate: ") + cudaGetErrorString(ce));
      }
    }
    while (err > tol && iters < max_sweeps) {
      DI_CK(cudaGraphLaunch(sweep_x, s));
      launches += per_sweep;
      DI_CK(cudaMemcpyAsync(part.data(), dacc, kGsBlocks * 8, cudaMemcpyDeviceToHost, s));
      DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
      DI_CK(cudaStreamSynchronize(s));
      double tot = 0.0;
      for (double p : part) tot += p;
      const double e = g.sc_host->e;
      err = tot * d / (1.0 - d - d * e);
      iters++;
    }
    cudaGraphExecDestroy(sweep_x);
    cudaGraphDestroy(sweep_g);
    dfree(dacc);
  }
  if (x != g.H) DI_CK(cudaMemcpyAsync(g.H, x, (size_t)n * 8, cudaMemcpyDeviceToDevice, s));
  DI_CK(cudaEventRecord(t1, s));
  DI_CK(cudaEventSynchronize(t1));
  DI_CK(cudaGetLastError());
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  g.solved = false;  // F/H no longer hold a D-iteration state: DI_RESUME is refused
  const bool conv = err <= tol;
  if (st) {
    memset(st, 0, sizeof(*st));
    st->sweeps = iters;
    st->link_diffusions = iters * g.l_global;
    st->nodes_scanned = iters * n;
    st->equivalent_iterations = (double)iters;
    st->gpu_launches = launches;
    st->solve_ms = ms;
    st->error_estimate = err;
    st->residual_l1 = err;
    st->converged = conv ? 1 : 0;
    st->variant = variant;
  }
  return conv ? DI_OK : DI_NOT_CONVERGED;
}

}  // namespace di
