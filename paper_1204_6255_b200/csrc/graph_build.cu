// graph_build.cu — device CSR/CSC builder (§2.1).
//
// The paper builds `vector<int> l_out[N]; vector<int> l_in[N]` on the host ("Init",
// timed separately). Here the link list is turned into a contiguous CSR in HBM:
//   key_k = src_k << b | dst_k  (b = bits(n))  -> radix sort -> optional drop of self-loops
//   and duplicates -> row_ptr by boundary scatter, col = low bits, deg, kloop.
// Everything is integer work and bit-exact (tests/test_gpu_build.py compares byte for byte
// with a numpy lexsort). The radix sort is CUB's (a library sort, like cuBLAS for a plain
// GEMM); every other step is a kernel below.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <cub/device/device_merge.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cub/cub.cuh>

#include "comm.cuh"
#include "di_common.cuh"

namespace di {
namespace {

// id validation (first bad link index) and, for the locality relabelling, in-degrees
// every id in [0, n); sources in [s_lo, s_hi) ([0, n), or the rank's range with DI_LOCAL_LINKS)
__global__ void k_validate(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                           int64_t L, int64_t n, int64_t s_lo, int64_t s_hi,
                           unsigned long long *__restrict__ bad, uint32_t *__restrict__ indeg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[k], t = dst[k];
    if (s < s_lo || s >= s_hi || t < 0 || t >= n)
      atomicMin(bad, (unsigned long long)k);
    else if (indeg)
      atomicAdd(indeg + t, 1u);
  }
}

// Pipelined host upload (one GPU, DESIGN.md §6 "upload"): the target ids arrive first and are
// validated (and counted for the relabelling) while the source ids are still being copied
__global__ void k_validate_dst(const int32_t *__restrict__ dst, int64_t L, int64_t n,
                               unsigned long long *__restrict__ bad, uint32_t *__restrict__ indeg,
                               int64_t k0) {   // (dst: the chunk starting at link k0)
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = dst[k];
    if (t < 0 || t >= n)
      atomicMin(bad, (unsigned long long)(k0 + k));
    else if (indeg)
      atomicAdd(indeg + t, 1u);
  }
}

// ... then every chunk of source ids, once copied: validated, and its (src, dst) keys made
// (k_make_keys' format; a link with a bad id gets key 0, the upload fails after the last chunk)
__global__ void k_make_keys_chunk(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                  int64_t k0, int64_t k1, int64_t n, int b,
                                  const int32_t *__restrict__ new_of, uint64_t *__restrict__ keys,
                                  unsigned long long *__restrict__ bad) {
  for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1;
       k += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = src[k], t = dst[k];
    if (s < 0 || s >= n) {
      atomicMin(bad, (unsigned long long)k);
      keys[k] = 0;
      continue;
    }
    if (t < 0 || t >= n) {   // (reported by k_validate_dst)
      keys[k] = 0;
      continue;
    }
    if (new_of) {
      s = new_of[s];
      t = new_of[t];
    }
    keys[k] = ((uint64_t)(uint32_t)s << b) | (uint64_t)(uint32_t)t;
  }
}

// rank r (0 = largest in-degree) -> internal id. The first hot[g] ranks of range g are placed
// contiguously at the range start (the replicated-accumulator targets of a skewed graph, async.cu);
// the others go to stripe r' % P at position r' / P (r' = r - hot), stripes laid out contiguously.
// Nodes of similar rank share L2 lines (hot lines are fully hot) while the P hottest sit in P
// different lines. P is a prime near (#nodes)/1024: a power-of-two stripe length would put all
// stripe heads (the hottest lines) at one power-of-two address stride, which the L2 slice hash
// maps onto fewer slices (C4: 16384 stripes 65.7 ms, 16411 63.1 ms). Multi-GPU: the sorted order
// is (owner range, rank) and every range is placed on its own, so a rank's internal ids stay in
// the node range it owns.
// Two-tier placement (graphs whose F exceeds the L2 several times, DESIGN.md §6 "cold bins"): the
// first tier[g] ranks after the hot ones fill the prefix [lo + hot, lo + hot + tier) — striped
// among themselves (stripes2 stripes) — so that "hot target" is the plain test j < cold_lo, and
// the remaining ranks are striped over the rest of the range.
// Line spread (option line_spread = G < 16): inside a stripe, position idx (0 = hottest) is not
// slot idx: groups of G consecutive positions are dealt round-robin over the stripe's lines of
// 16 nodes, so a line holds G nodes of similar rank (one 32-B sector for G = 4) and 16 / G rank
// classes. The hot set then spans 16 / G times more lines, and the L2 slices — each a hash of the
// line address — share its requests more evenly: with 16 hot nodes per line C4's hot traffic sits
// on ~50k lines (~300 per slice), and the busiest slice runs ~20 % above the average (ncu:
// lts__t_tag_requests max 95 %, avg 79 %; a random assignment of those lines gives the same).
struct PlaceParams {
  int64_t hot[kMaxWorld];
  int64_t stripes[kMaxWorld];
  int64_t tier[kMaxWorld];
  int64_t stripes2[kMaxWorld];
  int spread;   // nodes of one rank class per 16-node line (16: no spreading)
  int64_t warm; // range 0: warm ranks after the hot ones, one every 2^wshift ids (async.cu warm tier)
  int wshift;
};

__device__ __forceinline__ int64_t spread_slot(int64_t idx, int64_t len, int G) {
  const int64_t Q = len / 16;   // whole lines of the stripe (the tail stays in place)
  if (G >= 16 || idx >= 16 * Q) return idx;
  const int64_t t = idx / G, c = idx % G;
  return (t % Q) * 16 + (t / Q) * G + c;
}

__device__ __forceinline__ int64_t stripe_pos(int64_t q, int64_t m, int64_t P, int G) {
  if (P < 1) P = 1;
  if (P > m) P = m;
  const int64_t M = m / P, rem = m % P;
  const int64_t s = q % P, idx = q / P;
  const int64_t len = M + (s < rem ? 1 : 0);
  return s * M + (s < rem ? s : rem) + spread_slot(idx, len, G);
}

__global__ void k_place(const int32_t *__restrict__ sorted_old, int64_t n, DistBounds bd,
                        PlaceParams pp, int32_t *__restrict__ new_of, int32_t *__restrict__ old_of) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    int g = 0;
    while (g + 1 < bd.world && r >= bd.b[g + 1]) g++;
    const int64_t lo = bd.b[g], rr = r - lo, hot = pp.hot[g];
    const int64_t W = g == 0 ? pp.warm : 0;
    int64_t k;
    const int64_t tier = pp.tier[g] > 0 ? pp.tier[g] - W : 0;   // the first tier's non-warm ids
    if (rr < hot) {
      k = lo + rr;
    } else if (rr < hot + W) {      // warm ranks: offsets 0, S, 2S, ... after the hot ids
      k = lo + hot + ((rr - hot) << pp.wshift);
    } else {
      // c = offset among the non-warm ids after the hot ones, then skip the warm offsets
      const int64_t q2 = rr - W - hot;
      int64_t c;
      if (q2 < tier) {              // first tier: striped inside the prefix
        c = stripe_pos(q2, tier, pp.stripes2[g], pp.spread);
      } else {
        const int64_t m = bd.b[g + 1] - lo - hot - tier - W;
        c = tier + stripe_pos(q2 - tier, m, pp.stripes[g], pp.spread);
      }
      if (W > 0 && pp.wshift == 0) {   // warm ranks contiguous after the hot ones
        c += W;
      } else if (W > 0) {
        const int64_t S1 = (1ll << pp.wshift) - 1, kq = c / S1;
        c = kq < W ? c + kq + 1 : c + W;
      }
      k = lo + hot + c;
    }
    const int32_t o = sorted_old[r];
    new_of[o] = (int32_t)k;
    old_of[k] = o;
  }
}

int64_t prime_at_most(int64_t x) {
  if (x < 2) return 1;
  for (int64_t p = x; p >= 2; p--) {
    bool prime = true;
    for (int64_t d = 2; d * d <= p; d++)
      if (p % d == 0) {
        prime = false;
        break;
      }
    if (prime) return p;
  }
  return 1;
}

// relabelling key: (owner range of i, descending in-degree); ties keep ascending id (stable sort)
__global__ void k_perm_keys64(const uint32_t *__restrict__ indeg, int64_t n, DistBounds bd,
                              uint64_t *__restrict__ key, int32_t *__restrict__ iota) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int g = 0;
    while (g + 1 < bd.world && i >= bd.b[g + 1]) g++;
    key[i] = ((uint64_t)g << 32) | (uint64_t)(0xFFFFFFFFu - indeg[i]);
    iota[i] = (int32_t)i;
  }
}

// in-links of the K first ranks (the warm tier's candidates), one block
__global__ void k_topsum(const uint32_t *__restrict__ indeg, const int32_t *__restrict__ sorted, int64_t K,
                         unsigned long long *out) {
  __shared__ unsigned long long s[256];
  unsigned long long x = 0;
  for (int64_t r = threadIdx.x; r < K; r += blockDim.x) x += indeg[sorted[r]];
  s[threadIdx.x] = x;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// out-degree histogram in the caller's numbering (partition weights)
__global__ void k_outdeg(const int32_t *__restrict__ src, int64_t L, int64_t *__restrict__ od) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long *>(od + src[k]), 1ull);
}

// bound g = smallest i with 20*pre[i] + 12*i >= g * W / world (W = 20 L + 12 n): ranges balanced
// on the counted bytes of a full sweep (20 per link, 12 per scanned node)
__global__ void k_bounds(const int64_t *__restrict__ pre, int64_t n, int world, int64_t *out) {
  const int g = threadIdx.x;
  if (g > world) return;
  const double W = 20.0 * (double)pre[n] + 12.0 * (double)n;
  const double target = W * (double)g / (double)world;
  int64_t a = 0, b = n;  // answer in [0, n]
  while (a < b) {
    const int64_t m = (a + b) / 2;
    if (20.0 * (double)pre[m] + 12.0 * (double)m >= target) b = m; else a = m + 1;
  }
  out[g] = (g == 0) ? 0 : (g == world ? n : a);
}


__global__ void k_make_keys(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                            int64_t L, int b, const int32_t *__restrict__ new_of,
                            uint64_t *__restrict__ keys) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = src[k], t = dst[k];
    if (new_of) {
      s = new_of[s];
      t = new_of[t];
    }
    keys[k] = ((uint64_t)(uint32_t)s << b) | (uint64_t)(uint32_t)t;
  }
}

// keep[k]: not (drop_self and s == t) and not (dedup and key_k == key_{k-1})
// partitioned build: the keys of the links whose source this rank owns (caller's numbering
// [lo, hi)), appended in any order (the sort follows); one counter reservation per warp
__global__ void k_make_own_keys(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                                int64_t L, int b, int64_t lo, int64_t hi,
                                const int32_t *__restrict__ new_of, uint64_t *__restrict__ keys,
                                unsigned long long *count) {
  const int lane = threadIdx.x & 31;
  for (int64_t k0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; k0 < L;
       k0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = k0 + lane;
    int32_t s = 0, t = 0;
    bool own = false;
    if (k < L) {
      s = src[k];
      own = s >= lo && s < hi;
      if (own) t = dst[k];
    }
    const unsigned m = __ballot_sync(0xffffffffu, own);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (own) {
      if (new_of) {
        s = new_of[s];
        t = new_of[t];
      }
      keys[base + __popc(m & ((1u << lane) - 1))] =
          ((uint64_t)(uint32_t)s << b) | (uint64_t)(uint32_t)t;
    }
  }
}

__global__ void k_keep_flags(const uint64_t *__restrict__ keys, int64_t L, int b, int dedup,
                             int drop_self, uint8_t *__restrict__ keep) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = keys[k];
    bool ok = true;
    if (drop_self && (key >> b) == (key & mask)) ok = false;
    if (dedup && k > 0 && keys[k - 1] == key) ok = false;
    keep[k] = ok;
  }
}

// row_ptr[i] = first k with major(key_k) >= i; col[k] = minor(key_k); kloop via self entries.
// keys: the links of rows [lo, lo + n) (majors relative to lo); row ids of the output are local.
__global__ void k_csr_from_sorted(const uint64_t *__restrict__ keys, int64_t L, int64_t n, int b,
                                  int64_t lo, int64_t *__restrict__ ptr, int32_t *__restrict__ idx,
                                  int32_t *__restrict__ kloop) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= L;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t cur = (k < L) ? (int64_t)(keys[k] >> b) - lo : n;
    int64_t prev = (k > 0) ? (int64_t)(keys[k - 1] >> b) - lo : -1;
    for (int64_t i = prev + 1; i <= cur; i++) ptr[i] = k;
    if (k < L) {
      int32_t minor = (int32_t)(keys[k] & mask);
      idx[k] = minor;
      if (kloop && (int64_t)minor == cur + lo) atomicAdd(&kloop[cur], 1);
    }
  }
}

// ---- row-sort build (one GPU, links kept as given): instead of sorting 64-bit (src, dst) keys,
// a counting sort by source (out-degrees -> row offsets -> scatter) and a sort inside each row
// (CUB segmented sort). Out-degrees in the caller's numbering, counted during validation (links
// are often grouped by source: the lanes of a warp with the same source add once).
__global__ void k_outdeg_agg(const int32_t *__restrict__ src, int64_t L, uint32_t *__restrict__ od) {
  const int lane = threadIdx.x & 31;
  for (int64_t k0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; k0 < L;
       k0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = k0 + lane;
    const int32_t s = k < L ? src[k] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    if (s >= 0 && lane == __ffs(peers) - 1) atomicAdd(od + s, (uint32_t)__popc(peers));
  }
}

// out-degree of internal row k (the scan input of the row offsets)
__global__ void k_new_deg(const uint32_t *__restrict__ od, const int32_t *__restrict__ old_of,
                          int64_t n, int64_t *__restrict__ deg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    deg[k] = od[old_of ? old_of[k] : k];
  if (blockIdx.x == 0 && threadIdx.x == 0) deg[n] = 0;
}

// each link to the next free slot of its (internal) row; self-loops counted per row
__global__ void k_scatter_rows(const int32_t *__restrict__ src, const int32_t *__restrict__ dst,
                               int64_t L, const int32_t *__restrict__ new_of,
                               unsigned long long *__restrict__ cursor, int32_t *__restrict__ out,
                               int32_t *__restrict__ kloop) {
  const int lane = threadIdx.x & 31;
  for (int64_t k0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; k0 < L;
       k0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = k0 + lane;
    int32_t s = -1, t = 0;
    if (k < L) {
      s = src[k];
      t = dst[k];
      if (new_of) {
        s = new_of[s];
        t = new_of[t];
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (s >= 0 && lane == leader) base = atomicAdd(cursor + s, (unsigned long long)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (s >= 0) {
      out[base + __popc(peers & ((1u << lane) - 1))] = t;
      if (s == t) atomicAdd(kloop + s, 1);
    }
  }
}

// Rows sorted by target after the scatter (craw -> col), by size class (the CUB segmented sort
// took 33 ms on C4's 16.7M rows): rows of <= 16 links one thread each (insertion sort in
// registers/L1; rows of 0-1 links copied), 17-256 links one warp each (WarpMergeSort), 257-4096
// one block each (BlockRadixSort in shared memory), longer rows by a CUB segmented radix sort.
constexpr int kRsSmall = 16, kRsMid = 256, kRsBig = 4096;
__global__ void k_rowsort_small(const int64_t *__restrict__ ptr, int64_t n,
                                const int32_t *__restrict__ in, int32_t *__restrict__ out,
                                int32_t *__restrict__ mid, int32_t *__restrict__ big,
                                int32_t *__restrict__ huge, unsigned long long *__restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane; i0 < n;
       i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + lane;
    int64_t b = 0, len = -1;
    if (i < n) {
      b = ptr[i];
      len = ptr[i + 1] - b;
    }
    if (len >= 0 && len <= kRsSmall) {
      int32_t a[kRsSmall];
      for (int k = 0; k < len; k++) {
        const int32_t x = in[b + k];
        int m = k;
        while (m > 0 && a[m - 1] > x) {
          a[m] = a[m - 1];
          m--;
        }
        a[m] = x;
      }
      for (int k = 0; k < len; k++) out[b + k] = a[k];
    }
    // the longer rows into their class lists (one reservation per class and warp)
    const int cls = len <= kRsSmall ? -1 : (len <= kRsMid ? 0 : (len <= kRsBig ? 1 : 2));
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const unsigned m = __ballot_sync(0xffffffffu, cls == c);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == __ffs(m) - 1) base = atomicAdd(cnt + 16 * c, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
      if (cls == c) {
        int32_t *lst = c == 0 ? mid : (c == 1 ? big : huge);
        lst[base + __popc(m & ((1u << lane) - 1))] = (int32_t)i;
      }
    }
  }
}

__global__ void k_rowsort_mid(const int64_t *__restrict__ ptr, const int32_t *__restrict__ rows,
                              int64_t nrows, const int32_t *__restrict__ in, int32_t *__restrict__ out) {
  using WS = cub::WarpMergeSort<int32_t, kRsMid / 32, 32>;
  __shared__ typename WS::TempStorage ts[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)8 + warp;
  if (r >= nrows) return;
  const int64_t i = rows[r], b = ptr[i], len = ptr[i + 1] - b;
  int32_t k[kRsMid / 32];
#pragma unroll
  for (int u = 0; u < kRsMid / 32; u++) {   // blocked arrangement: lane owns 8 consecutive slots
    const int64_t p = (int64_t)lane * (kRsMid / 32) + u;
    k[u] = p < len ? in[b + p] : INT32_MAX;
  }
  WS(ts[warp]).Sort(k, [](int32_t x, int32_t y) { return x < y; });
#pragma unroll
  for (int u = 0; u < kRsMid / 32; u++) {
    const int64_t p = (int64_t)lane * (kRsMid / 32) + u;
    if (p < len) out[b + p] = k[u];
  }
}

__global__ void __launch_bounds__(256) k_rowsort_big(const int64_t *__restrict__ ptr,
                                                     const int32_t *__restrict__ rows, int bits,
                                                     const int32_t *__restrict__ in,
                                                     int32_t *__restrict__ out) {
  using BS = cub::BlockRadixSort<uint32_t, 256, kRsBig / 256>;
  __shared__ typename BS::TempStorage ts;
  const int64_t i = rows[blockIdx.x], b = ptr[i], len = ptr[i + 1] - b;
  uint32_t k[kRsBig / 256];
#pragma unroll
  for (int u = 0; u < kRsBig / 256; u++) {
    const int64_t p = (int64_t)threadIdx.x * (kRsBig / 256) + u;
    k[u] = p < len ? (uint32_t)in[b + p] : (1u << bits);   // padding sorts last
  }
  BS(ts).Sort(k, 0, bits + 1);
#pragma unroll
  for (int u = 0; u < kRsBig / 256; u++) {
    const int64_t p = (int64_t)threadIdx.x * (kRsBig / 256) + u;
    if (p < len) out[b + p] = (int32_t)k[u];
  }
}



__global__ void k_deg(const int64_t *__restrict__ ptr, int64_t n, int32_t *__restrict__ deg,
                      const int32_t *__restrict__ kloop, int *__restrict__ any_loop) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    deg[i] = (int32_t)(ptr[i + 1] - ptr[i]);
    if (kloop[i]) *any_loop = 1;
  }
}

__global__ void k_swap_keys(const uint64_t *__restrict__ in, int64_t L, int b,
                            uint64_t *__restrict__ out) {
  const uint64_t mask = (1ull << b) - 1;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < L;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = in[k];
    out[k] = ((key & mask) << b) | (key >> b);
  }
}

// option build_trace = 1: host timestamps of the build phases on stderr (diagnostics)
}  // namespace

void btrace(const char *what) {
  const bool on = options().build_trace != 0;
  if (!on) return;
  static thread_local std::chrono::steady_clock::time_point t0;
  const auto now = std::chrono::steady_clock::now();
  if (std::string(what) == "start") t0 = now;
  fprintf(stderr, "[di build] %-8s %8.2f ms\n", what,
          std::chrono::duration<double, std::milli>(now - t0).count());
}

namespace {

int grid_for(int64_t n, int sms) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// All temporaries of one build come from ONE pool allocation carved here (sizes known up front,
// CUB temp sizes queried with null pointers). One block of the same size per upload is reused by
// the stream-ordered pool without growing it; separate allocations of mixed sizes fragmented the
// pool and made some uploads map fresh memory (0.5 s on C4).
struct Arena {
  char *base = nullptr;
  size_t cap = 0, off = 0;
  ~Arena() {
    if (base) dfree(base);
  }
  static size_t up(size_t x) { return (x + 255) & ~(size_t)255; }
  template <typename T>
  T *take(size_t bytes) {
    T *p = reinterpret_cast<T *>(base + off);
    off += up(bytes ? bytes : 1);
    return p;
  }
};

}  // namespace

di_status build_graph(Graph &g, const int32_t *src, const int32_t *dst, int64_t L,
                      uint32_t flags) {
  cudaStream_t st = g.stream;
  const int64_t n = g.n_global;
  const int world = g.world;
  int b = 1;
  while ((1ll << b) < n) b++;
  const int sms = g.num_sms;
  const bool host = flags & DI_HOST_PTRS;
  const bool reorder = !(flags & DI_NO_REORDER);
  const int dedup = (flags & DI_DEDUP) ? 1 : 0, drop_self = (flags & DI_DROP_SELF_LOOPS) ? 1 : 0;
  const size_t LL = (size_t)(L > 0 ? L : 1);
  // one GPU, links kept as given, no CSC: counting sort by source + segmented sort of the rows
  const bool rowsort = g.row_sort && world == 1 && !dedup && !drop_self && !(flags & DI_BUILD_CSC) &&
                       L > 0;
  int wb = 0;
  while ((1 << wb) < world) wb++;
  // Pipelined host upload (one GPU, host link list, key sort): the target ids are copied first, and
  // while the source ids follow in kPipeChunks chunks the device validates the targets, counts the
  // in-degrees and relabels, then makes and sorts the keys of every chunk as soon as it has landed;
  // the sorted chunks are merged at the end. The PCIe copy (~55 GB/s: 39 ms for C4's 2.1 GB) then
  // hides most of the build (serial: copy, then 19 ms of relabelling, key sort and CSR).
  // (CUB's DeviceMerge counts are int and its output offsets overflow past 2^31 - 1 keys: longer
  //  lists, e.g. C5's 2.16e9 links, take the one-sort path)
  const bool pipe = host && world == 1 && !rowsort && L >= kPipeMinLinks && L <= (int64_t)INT32_MAX;
  const int64_t chunk = pipe ? (L + kPipeChunks - 1) / kPipeChunks : 0;

  btrace("start");
  // ---- one arena for every temporary: CUB temp sizes first (null pointers: size queries only)
  // (partitioned: the link keys, their sort and the compaction live in a second arena sized by
  //  this rank's own links, allocated once the partition is known)
  const bool part = world > 1;
  size_t cub_tmp = 0, q = 0;
  if (!part && !rowsort) {
    DI_CK(cub::DeviceRadixSort::SortKeys(nullptr, q, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                         (int64_t)LL, 0, 2 * b, st));
    cub_tmp = std::max(cub_tmp, q);
  }
  if (pipe) {
    DI_CK(cub::DeviceRadixSort::SortKeys(nullptr, q, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                         (int64_t)chunk, 0, 2 * b, st));
    cub_tmp = std::max(cub_tmp, q);
    DI_CK(cub::DeviceMerge::MergeKeys(nullptr, q, (const uint64_t *)nullptr, (int)(L / 2 + chunk),
                                      (const uint64_t *)nullptr, (int)(L / 2 + chunk), (uint64_t *)nullptr,
                                      cuda::std::less<uint64_t>{}, st));
    cub_tmp = std::max(cub_tmp, q);
  }
  constexpr int64_t kSegMax = 1ll << 30;   // items per segmented-sort call (its counts are int)
  if (rowsort) {
    DI_CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, q, (const int32_t *)nullptr,
                                                  (int32_t *)nullptr, (int)std::min<int64_t>(L, kSegMax),
                                                  (int)std::min<int64_t>(n, L / kRsBig + 1),
                                                  (const int32_t *)nullptr, (const int32_t *)nullptr, 0,
                                                  2 * b, st));
    cub_tmp = std::max(cub_tmp, q);
    DI_CK(cub::DeviceScan::ExclusiveSum(nullptr, q, (int64_t *)nullptr, (int64_t *)nullptr, n + 1,
                                        st));
    cub_tmp = std::max(cub_tmp, q);
  }
  if (!part && (dedup || drop_self)) {
    DI_CK(cub::DeviceSelect::Flagged(nullptr, q, (uint64_t *)nullptr, (uint8_t *)nullptr,
                                     (uint64_t *)nullptr, (int64_t *)nullptr, (int64_t)LL, st));
    cub_tmp = std::max(cub_tmp, q);
  }
  if (reorder) {
    DI_CK(cub::DeviceRadixSort::SortPairs(nullptr, q, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                          (int32_t *)nullptr, (int32_t *)nullptr, (int64_t)n, 0,
                                          32 + wb, st));
    cub_tmp = std::max(cub_tmp, q);
    DI_CK(cub::DeviceReduce::Max(nullptr, q, (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n,
                                 st));
    cub_tmp = std::max(cub_tmp, q);
  }
  if (world > 1) {
    DI_CK(cub::DeviceScan::ExclusiveSum(nullptr, q, (int64_t *)nullptr, (int64_t *)nullptr, n + 1,
                                        st));
    cub_tmp = std::max(cub_tmp, q);
  }
  const size_t nn = (size_t)n;
  size_t total = 0;
  auto add = [&](size_t x) { total += Arena::up(x ? x : 1); };
  if (host) {
    add(LL * 4);
    add(LL * 4);
  }
  if (!part && !rowsort) {
    add(LL * 8);                      // keys_a
    add(LL * 8);                      // keys_b
  }
  if (rowsort) {
    add(LL * 4);                      // rows before their sort
    add(nn * 4);                      // out-degrees (caller's numbering)
    add((nn + 1) * 8 + 1024);         // row degrees, the scatter cursors, then the row-class lists
  }
  add(cub_tmp);
  if (!part && (dedup || drop_self)) add(LL);    // keep flags (dedup / self-loops)
  add(64);                            // bad index / counts / max / key bounds
  add((kMaxWorld + 1) * 8);           // partition bounds
  if (reorder) {
    add(nn * 4);                      // indeg
    add(nn * 8);                      // relabel keys in/out
    add(nn * 8);
    add(nn * 4);                      // iota
    add(nn * 4);                      // sorted ranks
  }
  if (world > 1 && !g.local_links) add((nn + 1) * 8);   // out-degrees (partition bounds)
  if (world > 1 && !g.local_links) add((nn + 1) * 8);   // prefix
  Arena ar;
  DI_CK(dmalloc(&ar.base, total));
  ar.cap = total;

  const int32_t *s_dev = src, *d_dev = dst;
  // pipelined upload: the copies on their own stream, an event after the targets and after every
  // chunk of sources (the build's kernels stay on st and wait for them)
  struct PipeRes {
    cudaStream_t cp = nullptr;
    cudaEvent_t ev[2 * kPipeChunks] = {};   // target chunks, then source chunks
    ~PipeRes() {   // (before the arena is released: declared after it)
      if (cp) cudaStreamSynchronize(cp);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
      if (cp) cudaStreamDestroy(cp);
    }
  } pr;
  if (host) {
    int32_t *hs = ar.take<int32_t>(LL * 4), *hd = ar.take<int32_t>(LL * 4);
    if (pipe) {
      DI_CK(cudaStreamCreateWithFlags(&pr.cp, cudaStreamNonBlocking));
      for (auto &e : pr.ev) DI_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      for (int h = 0; h < 2; h++)   // the targets, then the sources, chunk by chunk
        for (int c = 0; c < kPipeChunks; c++) {
          const int64_t k0 = std::min<int64_t>(L, c * chunk), k1 = std::min<int64_t>(L, k0 + chunk);
          if (k1 > k0)
            DI_CK(cudaMemcpyAsync((h ? hs : hd) + k0, (h ? src : dst) + k0, (size_t)(k1 - k0) * 4,
                                  cudaMemcpyHostToDevice, pr.cp));
          DI_CK(cudaEventRecord(pr.ev[h * kPipeChunks + c], pr.cp));
        }
    } else if (L > 0) {
      DI_CK(cudaMemcpyAsync(hs, src, (size_t)L * 4, cudaMemcpyHostToDevice, st));
      DI_CK(cudaMemcpyAsync(hd, dst, (size_t)L * 4, cudaMemcpyHostToDevice, st));
    }
    s_dev = hs;
    d_dev = hd;
  }
  uint64_t *ka = (part || rowsort) ? nullptr : ar.take<uint64_t>(LL * 8);
  uint64_t *kb = (part || rowsort) ? nullptr : ar.take<uint64_t>(LL * 8);
  int32_t *craw = rowsort ? ar.take<int32_t>(LL * 4) : nullptr;
  uint32_t *odeg = rowsort ? ar.take<uint32_t>(nn * 4) : nullptr;
  int64_t *cursor = rowsort ? ar.take<int64_t>((nn + 1) * 8 + 1024) : nullptr;
  void *tmp = ar.take<char>(cub_tmp);
  uint8_t *keep = (!part && (dedup || drop_self)) ? ar.take<uint8_t>(LL) : nullptr;
  char *small = ar.take<char>(64);
  unsigned long long *badb = reinterpret_cast<unsigned long long *>(small);
  int64_t *nsel = reinterpret_cast<int64_t *>(small + 16);
  uint32_t *mx = reinterpret_cast<uint32_t *>(small + 24);
  int64_t *bnd = ar.take<int64_t>((kMaxWorld + 1) * 8);
  unsigned long long init_bad = ~0ull;
  DI_CK(cudaMemcpyAsync(badb, &init_bad, 8, cudaMemcpyHostToDevice, st));
  uint32_t *indeg = nullptr;
  if (reorder) {
    indeg = ar.take<uint32_t>(nn * 4);
    DI_CK(cudaMemsetAsync(indeg, 0, nn * 4, st));
  }
  const bool local = g.local_links;   // DI_LOCAL_LINKS: this rank's links, sources in its range
  const int64_t s_lo = local ? g.local_lo : 0, s_hi = local ? g.local_hi : n;
  // a range outside [0, n) fails on every rank, in the collective below
  const bool bad_range = local && !(s_lo >= 0 && s_lo < s_hi && s_hi <= n);
  if (pipe) {   // the targets, chunk by chunk as they land (the sources: below)
    for (int c = 0; c < kPipeChunks; c++) {
      const int64_t k0 = std::min<int64_t>(L, c * chunk), k1 = std::min<int64_t>(L, k0 + chunk);
      DI_CK(cudaStreamWaitEvent(st, pr.ev[c], 0));
      if (k1 > k0)
        k_validate_dst<<<grid_for(k1 - k0, sms), 256, 0, st>>>(d_dev + k0, k1 - k0, n, badb, indeg, k0);
    }
  } else if (L > 0 && !bad_range) {
    k_validate<<<grid_for(L, sms), 256, 0, st>>>(s_dev, d_dev, L, n, s_lo, s_hi, badb, indeg);
  }
  if (rowsort) {
    DI_CK(cudaMemsetAsync(odeg, 0, nn * 4, st));
    k_outdeg_agg<<<grid_for(L, sms), 256, 0, st>>>(s_dev, L, odeg);
  }
  unsigned long long bad = ~0ull;
  if (!pipe) {
    DI_CK(cudaMemcpyAsync(&bad, badb, 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
  }
  btrace("sync1");
  if (local) {  // every rank learns whether any rank failed (no rank may leave a collective)
    int64_t *flag = reinterpret_cast<int64_t *>(small + 48);
    const int64_t mine = (bad != ~0ull || bad_range) ? 1 : 0;
    DI_CK(cudaMemcpyAsync(flag, &mine, 8, cudaMemcpyHostToDevice, st));
    di_status cs = g.comm->allreduce_i64(flag, 1, st);
    if (cs != DI_OK) return cs;
    int64_t any = 0;
    DI_CK(cudaMemcpyAsync(&any, flag, 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    if (bad_range) {
      set_error("di_graph_upload: DI_LOCAL_LINKS needs 0 <= dist->lo < dist->hi <= n, got [" +
                std::to_string(s_lo) + ", " + std::to_string(s_hi) + ")");
      return DI_EINVAL;
    }
    if (any && bad == ~0ull) {
      set_error("di_graph_upload: another rank's link list or range failed validation "
                "(DI_LOCAL_LINKS)");
      return DI_EINVAL;
    }
  }
  auto report_bad = [&](unsigned long long bad) {
    int32_t sv = 0, dv = 0;
    if (host) {
      sv = src[bad];
      dv = dst[bad];
    } else {
      cudaMemcpy(&sv, src + bad, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(&dv, dst + bad, 4, cudaMemcpyDeviceToHost);
    }
    if (local && (sv < s_lo || sv >= s_hi) && sv >= 0 && sv < n)
      set_error("di_graph_upload: link " + std::to_string(bad) + " (" + std::to_string(sv) +
                " -> " + std::to_string(dv) + ") has a source outside this rank's range [" +
                std::to_string(s_lo) + ", " + std::to_string(s_hi) + ") (DI_LOCAL_LINKS)");
    else
      set_error("di_graph_upload: link " + std::to_string(bad) + " (" + std::to_string(sv) +
                " -> " + std::to_string(dv) + ") has a node id outside [0, " + std::to_string(n) +
                ")");
    return DI_EINVAL;
  };
  if (bad != ~0ull) return report_bad(bad);
  if (local && reorder) {  // in-degrees over every rank's links
    di_status cs = g.comm->allreduce_u32(indeg, n, st);
    if (cs != DI_OK) return cs;
  }
  // ---- multi-GPU: 1-D node ranges in the caller's numbering, balanced on counted sweep bytes
  //      (SURVEY §8(e)); every rank holds the full link list and computes the same bounds
  DistBounds &bd = g.bounds;
  bd.world = world;
  bd.b[0] = 0;
  bd.b[1] = n;
  int64_t *od = (world > 1 && !local) ? ar.take<int64_t>((nn + 1) * 8) : nullptr;
  const int64_t *pre_dev = nullptr;   // out-degree prefix in the caller's numbering (partitioned)
  if (local) {  // the ranges the callers chose: gathered, checked to tile [0, n) in rank order
    int64_t *rr = reinterpret_cast<int64_t *>(bnd);
    const int64_t mine[2] = {g.local_lo, g.local_hi};
    DI_CK(cudaMemcpyAsync(rr, mine, 16, cudaMemcpyHostToDevice, st));
    int64_t *all = reinterpret_cast<int64_t *>(tmp);
    di_status cs = g.comm->allgather(rr, all, 16, st);
    if (cs != DI_OK) return cs;
    std::vector<int64_t> h((size_t)2 * world);
    DI_CK(cudaMemcpyAsync(h.data(), all, 16 * (size_t)world, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    bool ok = h[0] == 0 && h[2 * (world - 1) + 1] == n;
    for (int r = 0; r < world; r++) {
      ok = ok && h[2 * r] < h[2 * r + 1];
      if (r > 0) ok = ok && h[2 * r] == h[2 * r - 1];
      bd.b[r] = h[2 * r];
    }
    bd.b[world] = n;
    if (!ok) {
      set_error("di_graph_upload: DI_LOCAL_LINKS ranges do not tile [0, n) in rank order");
      return DI_EINVAL;
    }
  } else if (world > 1) {
    int64_t *pre = ar.take<int64_t>((nn + 1) * 8);
    pre_dev = pre;
    DI_CK(cudaMemsetAsync(od, 0, (nn + 1) * 8, st));
    if (L > 0) k_outdeg<<<grid_for(L, sms), 256, 0, st>>>(s_dev, L, od);
    size_t cb = cub_tmp;
    DI_CK(cub::DeviceScan::ExclusiveSum(tmp, cb, od, pre, n + 1, st));
    k_bounds<<<1, 32, 0, st>>>(pre, n, world, bnd);
    DI_CK(cudaMemcpyAsync(bd.b, bnd, (size_t)(world + 1) * 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    btrace("sync2");
    // every range non-empty (n >= world is checked by the caller)
    for (int r = 1; r < world; r++) {
      if (bd.b[r] < bd.b[r - 1] + 1) bd.b[r] = bd.b[r - 1] + 1;
      if (bd.b[r] > n - (world - r)) bd.b[r] = n - (world - r);
    }
    bd.b[world] = n;
  }
  g.lo = bd.b[g.rank];
  g.hi = bd.b[g.rank + 1];
  g.n = g.hi - g.lo;
  // ---- locality relabelling: node ids sorted by descending in-degree inside
  //      each owner range, so the hot push targets share L2 lines; ranges keep their extent
  if (reorder) {
    uint64_t *kin = ar.take<uint64_t>(nn * 8), *kout = ar.take<uint64_t>(nn * 8);
    int32_t *vin = ar.take<int32_t>(nn * 4), *sorted = ar.take<int32_t>(nn * 4);
    DI_CK(dmalloc(&g.old_of, nn * 4));
    DI_CK(dmalloc(&g.new_of, nn * 4));
    k_perm_keys64<<<grid_for(n, sms), 256, 0, st>>>(indeg, n, bd, kin, vin);
    size_t pb = cub_tmp;
    DI_CK(cub::DeviceRadixSort::SortPairs(tmp, pb, kin, kout, vin, sorted, (int64_t)n, 0, 32 + wb,
                                          st));
    uint32_t top = 0;  // largest in-degree (DI_ASYNC decides on replicated hot accumulators)
    size_t mb = cub_tmp;
    DI_CK(cub::DeviceReduce::Max(tmp, mb, indeg, mx, (int64_t)n, st));
    DI_CK(cudaMemcpyAsync(&top, mx, 4, cudaMemcpyDeviceToHost, st));
    // in-links of the ranks a warm tier would take (auto size), for its on/off decision below
    const bool want_warm = !g.partitioned && g.warm_opt != 0;
    const int64_t wk = want_warm ? std::min<int64_t>(n, kHotRanks + (g.warm_opt > 0 ? g.warm_opt : warm_fit())) : 0;
    unsigned long long topw = 0;
    unsigned long long *tw = reinterpret_cast<unsigned long long *>(small + 32);
    if (wk > 0) {
      k_topsum<<<1, 256, 0, st>>>(indeg, sorted, wk, tw);
      DI_CK(cudaMemcpyAsync(&topw, tw, 8, cudaMemcpyDeviceToHost, st));
    }
    DI_CK(cudaStreamSynchronize(st));
    btrace("sync3");
    g.max_indeg = top;
    // skewed in-degrees (single GPU): the kHotRanks hottest nodes first (replicated accumulators;
    // hot rows that are also hubs are pushed as hub items, async.cu)
    bool skewed = !g.partitioned && g.hot_acc && L > 0 &&
                  (double)top > g.repl_share * (double)L && n > 4 * kHotRanks;
    g.hot_count = skewed ? kHotRanks : 0;
    // warm tier (k_cycle's shared-memory accumulators, async.cu): the warm_count ranks after the
    // hot ones, one every 2^warm_shift ids of the first tier (or of the rest of the range); auto:
    // as many as k_cycle's CTAs hold in shared memory at full occupancy (C4: 4032)
    const int64_t prefix = g.hot_count;
    // cold bins (single GPU, F several times the L2): a first tier of ~kColdHotL2 of the L2 in
    // nodes takes the prefix after the hot ids; targets beyond it are "cold" (async.cu)
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g.device);
    if (l2 <= 0) l2 = 126 << 20;
    g.l2_bytes = l2;
    int64_t tier = 0;
    if (!g.partitioned && g.cold_mode != 0 &&
        (g.cold_mode == 1 || (double)n * 8.0 > kColdF_L2 * (double)l2)) {
      tier = std::min<int64_t>(n - prefix, (int64_t)(kColdHotL2 * (double)l2 / 8.0));
      if (g.cold_tier > 0) tier = std::min<int64_t>(n - prefix, g.cold_tier);
      if (tier < 0) tier = 0;
    }
    g.cold_lo = (tier > 0 && prefix + tier < n) ? prefix + tier : n;
    {
      const int64_t w = g.warm_opt < 0 ? (int64_t)warm_fit() : (int64_t)g.warm_opt;
      // auto (option warm = -1): on when the candidates take at least kWarmShare of the links
      // (skewed or not), the graph has at least kWarmLinks links per warm slot of the cycle's grid
      // (the flush, grid x slots REDs per cycle, then stays a few % of a cycle's pushes), and not
      // with cold bins. Measured (profiles/r2/c4_ab_warm.txt): C4 (R-MAT, the first 4096 ranks
      // take 15 % of the links) 58.1 -> 52.9 ms; C3 (host blocks, Zipf targets, 7 %) 23.6 ->
      // 32.9 ms; C2 (10M links, 51 %) 3.4 -> 4.9 ms; C5 with cold bins 585 -> 640 ms. An explicit
      // count (warm > 0) turns it on whenever it fits (n >= 8 x (warm + hot), no cold bins).
      const bool warm_pays = g.warm_opt > 0 ||
                             (wk > 0 && (double)topw >= kWarmShare * (double)L &&
                              (double)L >= kWarmLinks * (double)cycle_warps(g) / 8.0 * (double)wk);
      g.warm_count = (warm_pays && !(g.cold_lo < n) && w > 0 && n >= 8 * (w + g.hot_count)) ? w : 0;
    }
    g.warm_shift = 0;
    if (g.warm_count > 0) {
      const int64_t region = g.cold_lo < n ? tier : n - prefix;
      // auto spacing: the warm ids span about the first eighth of the region (C4: every 512 ids).
      // Fluid pushed to a warm id waits in shared memory until the CTA leaves the cycle, so the
      // earlier the warm ids come in the cycle the less fluid waits (C4, 4032 warm ranks, one every
      // 2^11 / 2^10 / 2^9 / 2^8 / 2^7 ids: 57.4 / 55.7 / 52.9 / 55.0 / 54.1 ms; contiguous, their
      // long rows made the first tiles the stragglers of every cycle: 300 ms)
      while (((g.warm_count << (g.warm_shift + 1)) << 3) <= region) g.warm_shift++;
      if (g.warm_shift_opt > 0) {
        g.warm_shift = g.warm_shift_opt;
        while (g.warm_shift > 0 && (g.warm_count << g.warm_shift) > region) g.warm_shift--;
      }
      if ((g.warm_count << g.warm_shift) > region) g.warm_count = 0;
    }
    PlaceParams pp;
    pp.spread = g.line_spread;
    pp.warm = g.warm_count;
    pp.wshift = g.warm_shift;
    for (int r = 0; r < world; r++) {
      const int64_t m = bd.b[r + 1] - bd.b[r];
      pp.hot[r] = (r == 0) ? prefix : 0;
      pp.tier[r] = (r == 0 && g.cold_lo < n) ? tier : 0;
      // partitioned: the hot remote targets of every range first (compact remote accumulator,
      // dist.cu); the same on every rank (bounds, world and the L2 size of this GPU type)
      g.rtier[r] = 0;
      if (g.partitioned && g.remote_compact) {
        const int64_t want = g.remote_tier > 0 ? g.remote_tier
                                               : (int64_t)(kColdHotL2 * (double)l2 / 8.0 / world);
        g.rtier[r] = std::max<int64_t>(0, std::min<int64_t>(m, want));
        pp.tier[r] = g.rtier[r] < m ? g.rtier[r] : 0;
      }
      const int64_t wr = r == 0 ? pp.warm : 0;   // (warm ids sit inside the first tier if any)
      const int64_t t1 = pp.tier[r] > 0 ? pp.tier[r] - wr : 0;
      pp.stripes2[r] = prime_at_most(std::max<int64_t>(1, t1 >> 10));
      pp.stripes[r] = g.stripes > 0 ? (int64_t)g.stripes
                                     : prime_at_most(std::max<int64_t>(1, (m - pp.hot[r] - t1 - wr) >> 10));
    }
    k_place<<<grid_for(n, sms), 256, 0, st>>>(sorted, n, bd, pp, g.new_of, g.old_of);
    g.reordered = true;
  }
  // ---- partitioned: only this rank's links (sources in [lo, hi) of the caller's numbering; the
  //      relabelling keeps every range in place) get keys, in a second arena of ~L/G keys
  int64_t Ls = L;
  Arena ar2;
  if (part) {
    int64_t pe[2] = {0, 0};   // own links = out-degree prefix at the range ends
    if (!local) {
      DI_CK(cudaMemcpyAsync(&pe[0], pre_dev + g.lo, 8, cudaMemcpyDeviceToHost, st));
      DI_CK(cudaMemcpyAsync(&pe[1], pre_dev + g.hi, 8, cudaMemcpyDeviceToHost, st));
      DI_CK(cudaStreamSynchronize(st));
    }
    Ls = local ? L : pe[1] - pe[0];   // DI_LOCAL_LINKS: every link passed is this rank's
    const size_t LS = (size_t)(Ls > 0 ? Ls : 1);
    size_t t2 = 0;
    DI_CK(cub::DeviceRadixSort::SortKeys(nullptr, q, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                         (int64_t)LS, 0, 2 * b, st));
    t2 = std::max(t2, q);
    if (dedup || drop_self) {
      DI_CK(cub::DeviceSelect::Flagged(nullptr, q, (uint64_t *)nullptr, (uint8_t *)nullptr,
                                       (uint64_t *)nullptr, (int64_t *)nullptr, (int64_t)LS, st));
      t2 = std::max(t2, q);
    }
    DI_CK(dmalloc(&ar2.base, 2 * Arena::up(LS * 8) + Arena::up(t2) + Arena::up(LS) + 256));
    ka = ar2.take<uint64_t>(LS * 8);
    kb = ar2.take<uint64_t>(LS * 8);
    tmp = ar2.take<char>(t2);
    keep = ar2.take<uint8_t>(LS);
    cub_tmp = t2;
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(small + 48);
    DI_CK(cudaMemsetAsync(cnt, 0, 8, st));
    if (L > 0)
      k_make_own_keys<<<grid_for(L, sms), 256, 0, st>>>(s_dev, d_dev, L, b, g.lo, g.hi, g.new_of,
                                                        ka, cnt);
    btrace("sync4b");
  } else if (pipe) {
    // every chunk as it lands: its keys, then its sort (ka -> kb), then — binary-counter order —
    // the merges it completes: level 1 pairs kb -> ka, level 2 ka -> kb, level 3 kb -> ka, so the
    // merges of the first chunks run while the last ones are still on the wire
    static_assert((kPipeChunks & (kPipeChunks - 1)) == 0, "kPipeChunks: a power of two");
    for (int c = 0; c < kPipeChunks; c++) {
      const int64_t k0 = std::min<int64_t>(L, c * chunk), k1 = std::min<int64_t>(L, k0 + chunk);
      DI_CK(cudaStreamWaitEvent(st, pr.ev[kPipeChunks + c], 0));
      k_make_keys_chunk<<<grid_for(k1 - k0, sms), 256, 0, st>>>(s_dev, d_dev, k0, k1, n, b, g.new_of, ka, badb);
      size_t tb = cub_tmp;
      DI_CK(cub::DeviceRadixSort::SortKeys(tmp, tb, ka + k0, kb + k0, (int64_t)(k1 - k0), 0, 2 * b, st));
      int64_t span = chunk;
      for (int lvl = 0, idx = c; idx & 1; lvl++, idx >>= 1, span *= 2) {
        const int64_t a0 = (int64_t)(c + 1) * chunk - 2 * span, m = a0 + span;
        const int64_t e = std::min<int64_t>(L, a0 + 2 * span);
        uint64_t *in = (lvl % 2 == 0) ? kb : ka, *out = (lvl % 2 == 0) ? ka : kb;
        tb = cub_tmp;
        DI_CK(cub::DeviceMerge::MergeKeys(tmp, tb, in + a0, (int)(m - a0), in + m, (int)(e - m), out + a0,
                                          cuda::std::less<uint64_t>{}, st));
      }
    }
    constexpr int kLevels = __builtin_ctz(kPipeChunks);
    if (kLevels % 2 == 1) std::swap(ka, kb);   // the last level wrote ka: kb = the sorted keys
    DI_CK(cudaMemcpyAsync(&bad, badb, 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    btrace("pipe");
    if (bad != ~0ull) return report_bad(bad);
  } else if (L > 0 && !rowsort) {
    k_make_keys<<<grid_for(L, sms), 256, 0, st>>>(s_dev, d_dev, L, b, g.new_of, ka);
  }
  btrace("sync4");
  if (rowsort) {  // (bad ids were rejected above: every link is valid here)
    g.l_global = L;
    g.l = L;
    const int64_t nl = g.n;
    DI_CK(dmalloc(&g.row_ptr, ((size_t)nl + 1) * 8));
    DI_CK(dmalloc(&g.col, ((size_t)L + 8) * 4));   // +8: the push reads aligned int4 groups
    DI_CK(cudaMemsetAsync(g.col + L, 0, 8 * 4, st));
    DI_CK(dmalloc(&g.deg, (size_t)nl * 4));
    DI_CK(dmalloc(&g.kloop, (size_t)nl * 4));
    DI_CK(cudaMemsetAsync(g.kloop, 0, (size_t)nl * 4, st));
    k_new_deg<<<grid_for(nl, sms), 256, 0, st>>>(odeg, g.reordered ? g.old_of : nullptr, nl, cursor);
    size_t sb = cub_tmp;
    DI_CK(cub::DeviceScan::ExclusiveSum(tmp, sb, cursor, g.row_ptr, nl + 1, st));
    DI_CK(cudaMemcpyAsync(cursor, g.row_ptr, ((size_t)nl + 1) * 8, cudaMemcpyDeviceToDevice, st));
    if (options().build_trace) {
      cudaStreamSynchronize(st);
      btrace("rs_scan");
    }
    k_scatter_rows<<<grid_for(L, sms), 256, 0, st>>>(s_dev, d_dev, L, g.reordered ? g.new_of : nullptr,
                                                    reinterpret_cast<unsigned long long *>(cursor),
                                                    craw, g.kloop);
    // rows sorted by target (k_rowsort_*; the rows of more than kRsBig links: CUB segmented radix
    // sort, in calls of at most kSegMax links — its counts are int)
    {
      unsigned long long *cnt = reinterpret_cast<unsigned long long *>(cursor);   // reuse
      int32_t *lst_mid = reinterpret_cast<int32_t *>(cursor) + 128;
      int32_t *lst_big = lst_mid + nl;   // cursor holds (nl + 1) int64: room for 2 nl int32
      int32_t *lst_huge = reinterpret_cast<int32_t *>(odeg);   // out-degrees no longer needed
      DI_CK(cudaMemsetAsync(cnt, 0, 3 * 16 * 8, st));
      k_rowsort_small<<<grid_for(nl, sms), 256, 0, st>>>(g.row_ptr, nl, craw, g.col, lst_mid, lst_big,
                                                         lst_huge, cnt);
      if (options().build_trace) {
        cudaStreamSynchronize(st);
        btrace("rs_small");
      }
      unsigned long long hc[48];
      DI_CK(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
      DI_CK(cudaStreamSynchronize(st));
      const int64_t nmid = (int64_t)hc[0], nbig = (int64_t)hc[16], nhuge = (int64_t)hc[32];
      if (options().build_trace)
        fprintf(stderr, "[di build] rows: %lld mid, %lld big, %lld huge\n", (long long)nmid,
                (long long)nbig, (long long)nhuge);
      if (nmid > 0)
        k_rowsort_mid<<<(unsigned)((nmid + 7) / 8), 256, 0, st>>>(g.row_ptr, lst_mid, nmid, craw, g.col);
      if (options().build_trace) {
        cudaStreamSynchronize(st);
        btrace("rs_mid");
      }
      if (nbig > 0)
        k_rowsort_big<<<(unsigned)nbig, 256, 0, st>>>(g.row_ptr, lst_big, b, craw, g.col);
      if (options().build_trace) {
        cudaStreamSynchronize(st);
        btrace("rs_big");
      }

      if (nhuge > 0) {   // few rows: their offsets on the host, grouped into calls
        std::vector<int32_t> hr((size_t)nhuge);
        DI_CK(cudaMemcpyAsync(hr.data(), lst_huge, (size_t)nhuge * 4, cudaMemcpyDeviceToHost, st));
        std::vector<int64_t> rp((size_t)nl + 1);
        DI_CK(cudaMemcpyAsync(rp.data(), g.row_ptr, ((size_t)nl + 1) * 8, cudaMemcpyDeviceToHost, st));
        DI_CK(cudaStreamSynchronize(st));
        std::sort(hr.begin(), hr.end());
        std::vector<int32_t> ob, oe;
        int32_t *doff = lst_mid;   // the mid list is consumed (stream order): offsets go there
        size_t k = 0;
        while (k < hr.size()) {
          const int64_t base = rp[hr[k]];
          ob.clear();
          oe.clear();
          while (k < hr.size() && rp[hr[k] + 1] - base <= kSegMax) {
            ob.push_back((int32_t)(rp[hr[k]] - base));
            oe.push_back((int32_t)(rp[hr[k] + 1] - base));
            k++;
          }
          if (ob.empty()) return (set_error("di_graph_upload: a row of more than 2^30 links"), DI_EINVAL);
          const int ns = (int)ob.size();
          DI_CK(cudaMemcpyAsync(doff, ob.data(), (size_t)ns * 4, cudaMemcpyHostToDevice, st));
          DI_CK(cudaMemcpyAsync(doff + ns, oe.data(), (size_t)ns * 4, cudaMemcpyHostToDevice, st));
          size_t tb = cub_tmp;
          DI_CK(cub::DeviceSegmentedRadixSort::SortKeys(tmp, tb, craw + base, g.col + base,
                                                        (int)(oe.back()), ns, doff, doff + ns, 0, b + 1,
                                                        st));
          DI_CK(cudaStreamSynchronize(st));   // doff is reused by the next call
        }
      }
    }
    if (options().build_trace) {
      cudaStreamSynchronize(st);
      btrace("rs_sort");
    }
    int *any_loop = reinterpret_cast<int *>(small);
    DI_CK(cudaMemsetAsync(any_loop, 0, 4, st));
    k_deg<<<grid_for(nl, sms), 256, 0, st>>>(g.row_ptr, nl, g.deg, g.kloop, any_loop);
    int hl = 0;
    DI_CK(cudaMemcpyAsync(&hl, any_loop, 4, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    btrace("sync7");
    DI_CK(cudaGetLastError());
    g.has_loops = hl != 0;
    return DI_OK;
  }

  // ---- sort by (src, dst) (pipelined upload: done above)
  if (Ls > 0 && !pipe) {
    size_t tb = cub_tmp;
    DI_CK(cub::DeviceRadixSort::SortKeys(tmp, tb, ka, kb, (int64_t)Ls, 0, 2 * b, st));
  }
  // kb: sorted keys. Optional compaction.
  int64_t Lk = Ls;
  if (Ls > 0 && (dedup || drop_self)) {
    k_keep_flags<<<grid_for(Ls, sms), 256, 0, st>>>(kb, Ls, b, dedup, drop_self, keep);
    size_t sb = cub_tmp;
    DI_CK(cub::DeviceSelect::Flagged(tmp, sb, kb, keep, ka, nsel, (int64_t)Ls, st));
    DI_CK(cudaMemcpyAsync(&Lk, nsel, 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    btrace("sync5");
    std::swap(ka, kb);  // kb = compacted sorted keys
  }
  g.l_global = Lk;
  if (world > 1) {  // the global link count after dedup / self-loop removal: sum over the ranks
    int64_t *cnt = reinterpret_cast<int64_t *>(small + 48);
    DI_CK(cudaMemcpyAsync(cnt, &Lk, 8, cudaMemcpyHostToDevice, st));
    di_status cs = g.comm->allreduce_i64(cnt, 1, st);
    if (cs != DI_OK) return cs;
    DI_CK(cudaMemcpyAsync(&g.l_global, cnt, 8, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
  }
  // ---- this rank's rows: all of kb (partitioned) or everything (one GPU)
  const int64_t kbeg = 0, kend = Lk;
  const int64_t Ll = kend - kbeg;
  const int64_t nl = g.n;
  g.l = Ll;
  const size_t LlS = (size_t)(Ll > 0 ? Ll : 1);
  DI_CK(dmalloc(&g.row_ptr, ((size_t)nl + 1) * 8));
  // +8 elements of padding: the push reads whole aligned int4 groups around each row
  DI_CK(dmalloc(&g.col, (LlS + 8) * 4));
  DI_CK(cudaMemsetAsync(g.col + LlS, 0, 8 * 4, st));
  DI_CK(dmalloc(&g.deg, (size_t)nl * 4));
  DI_CK(dmalloc(&g.kloop, (size_t)nl * 4));
  DI_CK(cudaMemsetAsync(g.kloop, 0, (size_t)nl * 4, st));
  k_csr_from_sorted<<<grid_for(Ll + 1, sms), 256, 0, st>>>(kb + kbeg, Ll, nl, b, g.lo, g.row_ptr,
                                                          g.col, g.kloop);
  int *any_loop = reinterpret_cast<int *>(small);  // reuse (bad index no longer needed)
  DI_CK(cudaMemsetAsync(any_loop, 0, 4, st));
  k_deg<<<grid_for(nl, sms), 256, 0, st>>>(g.row_ptr, nl, g.deg, g.kloop, any_loop);
  int hl = 0;
  DI_CK(cudaMemcpyAsync(&hl, any_loop, 4, cudaMemcpyDeviceToHost, st));

  if (flags & DI_BUILD_CSC) {  // single GPU only (checked by the caller)
    if (Lk > 0) {
      k_swap_keys<<<grid_for(Lk, sms), 256, 0, st>>>(kb, Lk, b, ka);
      size_t sb = cub_tmp;
      DI_CK(cub::DeviceRadixSort::SortKeys(tmp, sb, ka, kb, (int64_t)Lk, 0, 2 * b, st));
    }
    const size_t LkS = (size_t)(Lk > 0 ? Lk : 1);
    DI_CK(dmalloc(&g.csc_ptr, ((size_t)n + 1) * 8));
    DI_CK(dmalloc(&g.csc_row, (LkS + 8) * 4));
    DI_CK(cudaMemsetAsync(g.csc_row + LkS, 0, 8 * 4, st));
    k_csr_from_sorted<<<grid_for(Lk + 1, sms), 256, 0, st>>>(kb, Lk, n, b, 0, g.csc_ptr,
                                                            g.csc_row, nullptr);
    g.has_csc = true;
  }
  DI_CK(cudaStreamSynchronize(st));
  btrace("sync7");
  DI_CK(cudaGetLastError());
  g.has_loops = hl != 0;
  return DI_OK;
}

}  // namespace di
