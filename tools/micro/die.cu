// Microbenchmark: does a fp64 RED cost more when the target's L2 home is on the other die?
// 1. probe: every SM times L2-hit loads to 64 reference 2 KB chunks -> SM die map (near/far split)
// 2. classify every 2 KB chunk of F by timing it from one SM per chunk (near -> that SM's die)
// 3. RED throughput: targets uniform / R-MAT-skewed, issued (a) from any SM, (b) only from SMs on
//    the target's home die, (c) only from the other die.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die die.cu
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ double ld_cg(const double *p) { double v; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }

// min latency (cycles) of dependent L2 loads to chunk c (2 KB = 256 doubles)
__device__ int chunk_lat(const double *F, long c) {
  const double *base = F + c * 256;
  double v = ld_cg(base);               // bring into L2
  long off = (long)v;                   // 0, creates a dependency
  int best = 1 << 30;
  for (int k = 0; k < 8; k++) {
    const double *p = base + off;       // same (now L2-resident) line every time
    long long t0 = clock64();
    double w = ld_cg(p);
    off += (long)w;
    long long t1 = clock64();
    int d = (int)(t1 - t0) + (int)off;
    best = d < best ? d : best;
  }
  return best;
}

// one CTA per SM (claimed by smid), 4 warps; lane 0 of each warp times a quarter of the chunks
__global__ void k_probe_all(const double *F, long nchunks, int *claimed, unsigned short *lat) {
  __shared__ int mine;
  if (threadIdx.x == 0) mine = atomicCAS(claimed + smid(), 0, 1) == 0;
  __syncthreads();
  if (!mine || (threadIdx.x & 31)) return;
  const unsigned s = smid();
  for (long c = threadIdx.x >> 5; c < nchunks; c += blockDim.x >> 5) lat[s * nchunks + c] = (unsigned short)chunk_lat(F, c);
}

__device__ __forceinline__ void red(double *p, double v) { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }

// MODE 0: one list, any SM.  MODE 1: SM on die d takes list d (local).  MODE 2: list 1-d (remote).
template <int MODE>
__global__ void k_red(double *F, const int *const *lists, const long *lens, int *ctr, const int *sm_die) {
  __shared__ long base;
  const int d = MODE == 0 ? 0 : (MODE == 1 ? sm_die[smid()] : 1 - sm_die[smid()]);
  const int *T = lists[d];
  const long len = lens[d];
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) base = (long)atomicAdd(ctr + d, 1) * 8192;
    __syncthreads();
    if (base >= len) return;
    for (long i = base + threadIdx.x; i < base + 8192 && i < len; i += blockDim.x) red(F + T[i], 1.0);
  }
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int lgn = 24; const long n = 1l << lgn;   // 134 MB of fp64, as C4's F
  double *F; CK(cudaMalloc(&F, n * 8)); CK(cudaMemset(F, 0, n * 8));
  const long nchunks = n / 256;
  // 1+2. every SM times every chunk; D(c) = mean latency from die-0 SMs - from die-1 SMs
  int *claimed; CK(cudaMalloc(&claimed, 4096)); CK(cudaMemset(claimed, 0, 4096));
  unsigned short *lat; CK(cudaMalloc(&lat, (size_t)sms * nchunks * 2));
  cudaEvent_t ea, eb; cudaEventCreate(&ea); cudaEventCreate(&eb); cudaEventRecord(ea);
  k_probe_all<<<sms * 8, 128>>>(F, nchunks, claimed, lat);
  cudaEventRecord(eb); CK(cudaEventSynchronize(eb)); float pms; cudaEventElapsedTime(&pms, ea, eb);
  std::vector<unsigned short> L((size_t)sms * nchunks); CK(cudaMemcpy(L.data(), lat, L.size() * 2, cudaMemcpyDeviceToHost));
  printf("probe %.1f ms\n", pms);
  // centre each chunk's column, then 2-cluster SMs: start from SM 0's sign pattern
  std::vector<float> Z((size_t)sms * nchunks);
  for (long c = 0; c < nchunks; c++) {
    double m = 0; for (int s = 0; s < sms; s++) m += L[s * nchunks + c]; m /= sms;
    for (int s = 0; s < sms; s++) Z[s * nchunks + c] = L[s * nchunks + c] - m;
  }
  std::vector<int> die(sms, 0);
  std::vector<double> D(nchunks);
  std::vector<float> w(Z.begin(), Z.begin() + nchunks);   // direction: SM 0's centred vector
  for (int it = 0; it < 6; it++) {
    for (int s = 0; s < sms; s++) { double dot = 0; for (long c = 0; c < nchunks; c++) dot += (double)Z[s * nchunks + c] * w[c]; die[s] = dot > 0 ? 0 : 1; }
    for (long c = 0; c < nchunks; c++) {
      double a = 0, b = 0; int na = 0, nb = 0;
      for (int s = 0; s < sms; s++) (die[s] ? (b += L[s * nchunks + c], nb++) : (a += L[s * nchunks + c], na++));
      D[c] = (na ? a / na : 0) - (nb ? b / nb : 0);
      w[c] = (float)D[c];
    }
  }
  int n0 = std::count(die.begin(), die.end(), 0);
  printf("SM die split %d / %d\ndie map:", n0, sms - n0); for (int s = 0; s < sms; s++) printf("%d", die[s]); printf("\n");
  int hist[40] = {0};
  for (long c = 0; c < nchunks; c++) { int b = (int)((D[c] + 40) / 2); b = b < 0 ? 0 : b > 39 ? 39 : b; hist[b]++; }
  printf("hist of D(c) = mean lat die0 SMs - die1 SMs, 2-cycle bins from -40:\n");
  for (int b = 0; b < 40; b++) printf("%d:%d ", -40 + 2 * b, hist[b]); printf("\n");
  std::vector<int> cdie[1]; cdie[0].resize(nchunks);
  long amb = 0, d0c = 0;
  for (long c = 0; c < nchunks; c++) { cdie[0][c] = D[c] < 0 ? 0 : 1; amb += std::fabs(D[c]) < 6; d0c += D[c] < 0; }
  printf("die0 chunks %ld / %ld, |D| < 6: %ld\n", d0c, nchunks, amb);
  // first-chunk reference: does the reference set match the classification?
  // 3. RED throughput
  int *sm_die; CK(cudaMalloc(&sm_die, sms * 4)); CK(cudaMemcpy(sm_die, die.data(), sms * 4, cudaMemcpyHostToDevice));
  const long ops = 1l << 27;
  std::mt19937_64 rng(1);
  for (int skew = 0; skew < 3; skew++) {
    std::vector<int> t_all(ops), t_d[2];
    std::vector<uint32_t> perm(n); std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::uniform_real_distribution<double> U(0, 1);
    for (long i = 0; i < ops; i++) {
      uint32_t j;
      if (skew == 0) j = rng() & (n - 1);
      else if (skew == 2) j = rng() & ((n >> 2) - 1);
      else { j = 0; for (int bit = 0; bit < lgn; bit++) j |= (U(rng) < 0.24 ? 1u : 0u) << bit; j = perm[j]; }
      t_all[i] = j;
      t_d[cdie[0][j >> 8]].push_back(j);
    }
    // equalise: each per-die list gets ops/2 entries (resample with wrap)
    for (int d = 0; d < 2; d++) { size_t m = t_d[d].size(); t_d[d].resize(ops / 2); for (size_t i = m; i < (size_t)ops / 2; i++) t_d[d][i] = t_d[d][i % m]; }
    int *dA, *d0, *d1; CK(cudaMalloc(&dA, ops * 4)); CK(cudaMalloc(&d0, ops * 2)); CK(cudaMalloc(&d1, ops * 2));
    CK(cudaMemcpy(dA, t_all.data(), ops * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d0, t_d[0].data(), ops * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d1, t_d[1].data(), ops * 2, cudaMemcpyHostToDevice));
    const int *hl[2]; long hlen[2];
    int **lists; long *lens; int *ctr; CK(cudaMalloc(&lists, 16)); CK(cudaMalloc(&lens, 16)); CK(cudaMalloc(&ctr, 8));
    const char *names[] = {"any SM", "home die", "other die"};
    for (int mode = 0; mode < 3; mode++) {
      if (mode == 0) { hl[0] = dA; hl[1] = dA; hlen[0] = hlen[1] = ops; }
      else { hl[0] = d0; hl[1] = d1; hlen[0] = hlen[1] = ops / 2; }
      CK(cudaMemcpy(lists, hl, 16, cudaMemcpyHostToDevice)); CK(cudaMemcpy(lens, hlen, 16, cudaMemcpyHostToDevice));
      float best = 1e9;
      for (int rep = 0; rep < 3; rep++) {
        CK(cudaMemset(ctr, 0, 8));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a);
        if (mode == 0) k_red<0><<<sms * 8, 256>>>(F, lists, lens, ctr, sm_die);
        if (mode == 1) k_red<1><<<sms * 8, 256>>>(F, lists, lens, ctr, sm_die);
        if (mode == 2) k_red<2><<<sms * 8, 256>>>(F, lists, lens, ctr, sm_die);
        cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
      }
      printf("%s targets, REDs from %-9s: %7.1f G/s\n", skew == 1 ? "R-MAT 134MB" : skew == 0 ? "uniform 134MB" : "uniform 34MB", names[mode], ops / (best * 1e-3) / 1e9);
    }
    cudaFree(dA); cudaFree(d0); cudaFree(d1);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
