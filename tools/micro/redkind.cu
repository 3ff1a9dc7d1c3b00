// Microbenchmark: L2 RED throughput by operand type and issue pattern, random targets in an
// L2-resident array (33.6 MB) and in a C4-sized one (134 MB).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o redkind redkind.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void k(void *A, uint32_t mask, int64_t ops, uint32_t seed) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ops; t += T * (MODE == 5 ? 4 : 1)) {
    if (MODE == 5) {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        uint32_t j = hash32((uint32_t)(t + u * T) * 2654435761u + seed) & mask;
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"((double *)A + j), "d"(1.0) : "memory");
      }
      continue;
    }
    uint32_t j = hash32((uint32_t)t * 2654435761u + seed) & mask;
    if (MODE == 0) asm volatile("red.global.add.f64 [%0], %1;" ::"l"((double *)A + j), "d"(1.0) : "memory");
    if (MODE == 1) asm volatile("red.global.add.u64 [%0], %1;" ::"l"((unsigned long long *)A + j), "l"(1ull) : "memory");
    if (MODE == 2) asm volatile("red.global.add.u32 [%0], %1;" ::"l"((unsigned *)A + 2 * j), "r"(1u) : "memory");
    if (MODE == 3) asm volatile("red.global.add.f32 [%0], %1;" ::"l"((float *)A + 2 * j), "f"(1.0f) : "memory");
    if (MODE == 4) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"((double *)A + j), "d"(1.0) : "memory");
    if (MODE == 6) asm volatile("st.global.f64 [%0], %1;" ::"l"((double *)A + j), "d"(1.0) : "memory");
  }
}

int main() {
  void *A; cudaMalloc(&A, (size_t)1 << 28); cudaMemset(A, 0, (size_t)1 << 28);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int64_t ops = 1ll << 28;
  const char *names[] = {"red.add.f64", "red.add.u64", "red.add.u32 (8B stride)", "red.add.f32 (8B stride)",
                         "red.relaxed.gpu.f64", "red.add.f64 x4 unrolled", "st.global.f64 (scatter)"};
  for (int lg : {22, 24}) {
    for (int mode = 0; mode < 7; mode++) {
      for (int occ : {4, 8}) {
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
          uint32_t mask = (1u << lg) - 1;
          cudaEventRecord(a);
          switch (mode) {
            case 0: k<0><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 1: k<1><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 2: k<2><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 3: k<3><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 4: k<4><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 5: k<5><<<sms * occ, 256>>>(A, mask, ops, rep); break;
            case 6: k<6><<<sms * occ, 256>>>(A, mask, ops, rep); break;
          }
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("%-26s array %6.1f MB, %d CTAs/SM: %7.1f Gop/s\n", names[mode], 8.0 * (1u << lg) / 1e6, occ, ops / (best * 1e-3) / 1e9);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
