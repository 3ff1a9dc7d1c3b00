// Microbenchmark: random fp64 RED / gather throughput on B200 vs target-array size.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomics atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }

template <int MODE>
__global__ void k(double *F, uint32_t mask, int64_t ops, uint32_t seed, double *sink) {
  const uint64_t pol = pol_last();
  double acc = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ops; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t j = hash32((uint32_t)t * 2654435761u + seed) & mask;
    if (MODE == 0) asm volatile("red.global.add.f64 [%0], %1;" :: "l"(F + j), "d"(1.0) : "memory");
    if (MODE == 1) asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(F + j), "d"(1.0), "l"(pol) : "memory");
    if (MODE == 2) acc += __ldg(F + j);
    if (MODE == 3) { // skewed: 80% of ops to the first 1/32 of the array
      uint32_t h = hash32(j ^ 0x9e37u);
      uint32_t jj = (h % 10 < 8) ? (j & (mask >> 5)) : j;
      asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(F + jj), "d"(1.0), "l"(pol) : "memory");
    }
  }
  if (MODE == 2 && acc == 12345.0) *sink = acc;
}

int main() {
  double *F, *sink; cudaMalloc(&F, (size_t)1 << 30); cudaMalloc(&sink, 8);
  cudaMemset(F, 0, (size_t)1 << 30);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int64_t ops = 1ll << 28;
  const char *names[] = {"red", "red_evict_last", "gather", "red_skew80"};
  for (int mode = 0; mode < 4; mode++) {
    for (int lg = 20; lg <= 27; lg++) {   // array of 2^lg doubles: 8 MB .. 1 GB
      uint32_t mask = (1u << lg) - 1;
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<sms * 8, 256>>>(F, mask, ops, rep, sink);
        if (mode == 1) k<1><<<sms * 8, 256>>>(F, mask, ops, rep, sink);
        if (mode == 2) k<2><<<sms * 8, 256>>>(F, mask, ops, rep, sink);
        if (mode == 3) k<3><<<sms * 8, 256>>>(F, mask, ops, rep, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 1) printf("%-16s array %7.1f MB : %7.1f Gop/s\n", names[mode], (8.0 * (1u << lg)) / 1e6, ops / (ms * 1e-3) / 1e9);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
