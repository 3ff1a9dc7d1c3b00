/* digen/gen_gpu.cu — per-source-range R-MAT + repair generation on the GPU (input plumbing only).
 *
 * The same recipe, hash and relabelling as digen/gen.c (R-MAT + repair, DESIGN.md "Input
 * recipe"), restricted to the links whose SOURCE lies in [lo, hi): every candidate e and every
 * repair draw is the same counter-based hash of (seed, tag, index), so each rank of a partitioned
 * run draws exactly its share of the link list that gen.c produces for the whole graph, without
 * materialising the rest (C5: 2.16e9 links, ~270e6 per rank at G = 8). Tested for equality with
 * gen.c (tests/test_gpu_digen.py).
 *
 * This module holds none of the D-iteration arithmetic; it shares no code with the product
 * (paper_1204_6255_b200/) or the oracle (oracle/). Output: unsorted packed keys
 * (src << 32 | dst), duplicates and raw self-loops included; the caller sorts, deduplicates and
 * drops self-loops (digen/__init__.py: rmat_range), which is gen.c's finish().
 *
 * Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared
 */
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

struct Params {
  int64_t n, m;
  int s;
  uint64_t seed;
  uint32_t A, AB, ABC;
  int half;
  uint64_t mask, key;
  double p_dang, p_zin_cond, p_chain_win;
  int repair, repair_in;
  int64_t lo, hi;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t h4(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ (tag << 56)) ^ a) + b);
}
__device__ __forceinline__ double u01(uint64_t h) {
  return __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0);
}
__device__ __forceinline__ uint64_t feistel(const Params &p, uint64_t x) {
  uint64_t L = (x >> p.half) & p.mask, R = x & p.mask;
  for (int r = 0; r < 4; r++) {
    const uint64_t t = L ^ (mix64(R ^ (p.key + (uint64_t)r * 0x9E37ULL)) & p.mask);
    L = R;
    R = t;
  }
  return (L << p.half) | R;
}
__device__ __forceinline__ int64_t perm_apply(const Params &p, int64_t x) {
  uint64_t y = (uint64_t)x;
  do {
    y = feistel(p, y);
  } while (y >= (uint64_t)p.n);
  return (int64_t)y;
}
// one R-MAT candidate of stream `tag`: raw (un-relabelled) endpoints; false if rejected (>= n)
__device__ __forceinline__ bool rmat_draw(const Params &p, uint64_t tag, uint64_t e, int64_t *src,
                                          int64_t *dst) {
  uint64_t s = 0, d = 0, h = 0;
  const uint64_t base = mix64(mix64(p.seed ^ (tag << 56)) ^ e);
  for (int l = 0; l < p.s; l++) {
    if ((l & 1) == 0) h = mix64(base + (uint64_t)(l >> 1));
    const uint32_t u = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
    int rb, cb;
    if (u < p.A) { rb = 0; cb = 0; }
    else if (u < p.AB) { rb = 0; cb = 1; }
    else if (u < p.ABC) { rb = 1; cb = 0; }
    else { rb = 1; cb = 1; }
    s = (s << 1) | (uint64_t)rb;
    d = (d << 1) | (uint64_t)cb;
  }
  if (s >= (uint64_t)p.n || d >= (uint64_t)p.n) return false;
  *src = (int64_t)s;
  *dst = (int64_t)d;
  return true;
}
__device__ __forceinline__ bool chain_info(const Params &p, int64_t x, bool *is_member) {
  *is_member = false;
  if (p.p_chain_win <= 0) return false;
  const int64_t w = x >> 3, off = x & 7;
  const uint64_t h = h4(p.seed, 'C', (uint64_t)w, 0);
  if (u01(h) >= p.p_chain_win) return false;
  const int len = 2 + (int)((h >> 3) % 3);
  if ((w << 3) + len >= p.n) return false;
  if (off == 0) return true;
  if (off <= len) {
    *is_member = true;
    return true;
  }
  return false;
}
__device__ __forceinline__ bool is_dangling(const Params &p, int64_t x) {
  bool mb;
  if (chain_info(p, x, &mb)) return false;
  return u01(h4(p.seed, 'D', (uint64_t)x, 0)) < p.p_dang;
}
__device__ __forceinline__ bool is_receiver(const Params &p, int64_t x) {
  bool mb;
  if (chain_info(p, x, &mb)) return false;
  if (u01(h4(p.seed, 'D', (uint64_t)x, 0)) < p.p_dang) return true;
  return !(u01(h4(p.seed, 'Z', (uint64_t)x, 0)) < p.p_zin_cond);
}

__device__ __forceinline__ void emit(uint64_t *out, int64_t cap, unsigned long long *cnt, int64_t s,
                                     int64_t d) {
  const unsigned long long pos = atomicAdd(cnt, 1ull);
  if ((int64_t)pos < cap) out[pos] = ((uint64_t)s << 32) | (uint64_t)(uint32_t)d;
}

__global__ void k_cands(Params p, uint64_t *out, int64_t cap, unsigned long long *cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < p.m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s, d;
    if (!rmat_draw(p, 'R', (uint64_t)e, &s, &d)) continue;
    s = perm_apply(p, s);
    if (s < p.lo || s >= p.hi) continue;
    d = perm_apply(p, d);
    if (p.repair && is_dangling(p, s)) continue;
    if (p.repair && !is_receiver(p, d)) continue;
    emit(out, cap, cnt, s, d);
  }
}

__global__ void k_repairs(Params p, uint64_t *out, int64_t cap, unsigned long long *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool mb;
    if (chain_info(p, i, &mb) && mb && i - 1 >= p.lo && i - 1 < p.hi) emit(out, cap, cnt, i - 1, i);
    if (i >= p.lo && i < p.hi && !is_dangling(p, i)) {  // step 4: guaranteed out-link
      for (uint64_t t = 0; t < 4096; t++) {
        int64_t s, d;
        if (!rmat_draw(p, 'O', ((uint64_t)i << 12) | t, &s, &d)) continue;
        d = perm_apply(p, d);
        if (d == i || !is_receiver(p, d)) continue;
        emit(out, cap, cnt, i, d);
        break;
      }
    }
    if (p.repair_in && is_receiver(p, i)) {  // step 5: guaranteed in-link (kept if its source is ours)
      for (uint64_t t = 0; t < 4096; t++) {
        int64_t s, d;
        if (!rmat_draw(p, 'I', ((uint64_t)i << 12) | t, &s, &d)) continue;
        s = perm_apply(p, s);
        if (s == i || is_dangling(p, s)) continue;
        if (s >= p.lo && s < p.hi) emit(out, cap, cnt, s, i);
        break;
      }
    }
  }
}

uint32_t thr32(double x) {
  const double v = __builtin_floor(x * 4294967296.0 + 0.5);
  if (v >= 4294967295.0) return 0xFFFFFFFFu;
  if (v <= 0) return 0;
  return (uint32_t)v;
}

}  // namespace

extern "C" {

/* Links of the R-MAT + repair graph (gen.c digen_rmat with the same arguments) whose source lies
 * in [lo, hi), as packed keys src << 32 | dst in `out` (device, capacity `cap`), unsorted, with
 * duplicates and raw self-loops. *count (host) = links drawn; if > cap, only cap were written and
 * the caller retries with a larger buffer. Enqueued on `stream` and synchronised. Returns 0, or
 * -1 on bad arguments, -3 on a CUDA error. */
int digen_rmat_range_gpu(int64_t n, int64_t m, double a, double b, double c, uint64_t seed,
                         double p_dangling, double p_zero_in, double chain_heads, int repair,
                         int repair_in, int64_t lo, int64_t hi, uint64_t *out, int64_t cap,
                         int64_t *count, void *stream) {
  if (n < 1 || n > 2147483647LL || m < 0 || lo < 0 || hi < lo || hi > n || !count) return -1;
  Params p;
  p.n = n;
  p.m = m;
  int s = 0;
  while ((1LL << s) < n) s++;
  p.s = s;
  p.seed = seed;
  p.A = thr32(a);
  p.AB = thr32(a + b);
  p.ABC = thr32(a + b + c);
  /* Feistel key and half width: gen.c perm_make(n, seed) */
  p.half = (s + 1) / 2;
  if (p.half == 0) p.half = 1;
  p.mask = (1ULL << p.half) - 1;
  {
    uint64_t z = seed ^ 0x5045524dULL;
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    p.key = z ^ (z >> 31);
  }
  p.repair = repair;
  p.p_dang = repair ? p_dangling : 0.0;
  p.p_zin_cond = (repair && p_dangling < 1.0) ? p_zero_in / (1.0 - p_dangling) : 0.0;
  p.p_chain_win = repair ? chain_heads * 8.0 : 0.0;
  p.repair_in = repair && repair_in;
  p.lo = lo;
  p.hi = hi;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *cnt = nullptr;
  if (cudaMallocAsync(&cnt, 8, st) != cudaSuccess) return -3;
  cudaMemsetAsync(cnt, 0, 8, st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_cands<<<sms * 8, 256, 0, st>>>(p, out, cap, cnt);
  if (repair) k_repairs<<<sms * 8, 256, 0, st>>>(p, out, cap, cnt);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(cnt, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -3;
  if (cudaGetLastError() != cudaSuccess) return -3;
  *count = (int64_t)h;
  return 0;
}

}  // extern "C"
