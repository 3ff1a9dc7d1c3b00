// Microbenchmark: R-MAT-skewed fp64 REDs into an L2-resident array; does replicating the hottest
// targets (kCopies copies, chosen by warp) lift the rate? (C4's top node takes ~0.09 % of links)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hot hot.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%d %s\n", __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

// targets < 0 encode hot slot -(h+1); the copy is chosen by global warp id
__global__ void k_red(double *F, double *rep, int copies, int nhot, int stride, const int *T, long len) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int copy = wid % copies;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < len; i += (long)gridDim.x * blockDim.x) {
    int j = T[i];
    double *p = j >= 0 ? F + j : rep + ((long)copy * nhot + (-j - 1)) * stride;
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(1.0) : "memory");
  }
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int lgn : {22, 24}) {
    const long n = 1l << lgn;
    const long ops = 1l << 27;
    double *F, *rep; CK(cudaMalloc(&F, n * 8)); CK(cudaMalloc(&rep, 64l * 512 * 16 * 8));
    CK(cudaMemset(F, 0, n * 8)); CK(cudaMemset(rep, 0, 64l * 512 * 16 * 8));
    std::mt19937_64 rng(7);
    std::vector<uint32_t> perm(1l << 24); std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<int> T(ops);
    std::vector<long> cnt(n, 0);
    const uint64_t thr = (uint64_t)(0.24 * 18446744073709551616.0);
    for (long i = 0; i < ops; i++) {
      uint32_t j = 0;
      for (int b = 0; b < 24; b++) j |= (rng() < thr ? 1u : 0u) << b;
      j = perm[j] & (n - 1);
      T[i] = j; cnt[j]++;
    }
    std::vector<int> order(n); std::iota(order.begin(), order.end(), 0);
    std::partial_sort(order.begin(), order.begin() + 512, order.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
    printf("n=2^%d: top target share %.4f %%, top-64 share %.3f %%\n", lgn, 100.0 * cnt[order[0]] / ops,
           100.0 * std::accumulate(order.begin(), order.begin() + 64, 0.0, [&](double s, int k) { return s + cnt[k]; }) / ops);
    int *dT; CK(cudaMalloc(&dT, ops * 4));
    for (int nhot : {0, 1, 8, 32, 64, 256}) {
      std::vector<int> slot(n, -1);
      for (int h = 0; h < nhot; h++) slot[order[h]] = h;
      std::vector<int> T2(T);
      for (long i = 0; i < ops; i++) if (slot[T2[i]] >= 0) T2[i] = -(slot[T2[i]] + 1);
      CK(cudaMemcpy(dT, T2.data(), ops * 4, cudaMemcpyHostToDevice));
      for (int copies : {1, 4, 16, 64}) for (int stride : {1, 4, 16}) {
        if (nhot == 0 && (copies > 1 || stride > 1)) continue;
        float best = 1e9;
        for (int rep_ = 0; rep_ < 3; rep_++) {
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a);
          k_red<<<sms * 8, 256>>>(F, rep, copies, nhot, stride, dT, ops);
          cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b);
          best = std::min(best, ms);
        }
        printf("  hot %3d copies %2d stride %2d: %6.1f G REDs/s\n", nhot, copies, stride, ops / (best * 1e-3) / 1e9);
      }
    }
    cudaFree(F); cudaFree(rep); cudaFree(dT);
  }
  return 0;
}
