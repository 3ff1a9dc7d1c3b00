// comm.cuh — the two collectives the partitioned sweep needs, behind one
// interface with two backends:
//   NcclComm  — one process per GPU, NCCL over NVLink/NVSwitch (libnccl.so.2 is dlopen'ed at
//               run time: the copy torch already loaded, so there is exactly one NCCL in the
//               process, and libdi.so still loads on a box without NCCL);
//   GroupComm — G ranks driven by G host threads of one process on one GPU ("emulated ranks":
//               the only way to run the multi-rank protocol with a single GPU). Ranks meet at a
//               host barrier; data moves with device-to-device copies. No kernel ever waits for
//               another rank's kernel (B200_PROFILING.md: never spin across ranks on one GPU).
// Both are called from the host sweep loop in dist.cu; every rank makes the same calls in the
// same order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "di_common.cuh"

namespace di {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  // in-place sums of small device arrays (every rank gets the same result, summed in rank order
  // for the group backend, NCCL's order for NCCL)
  virtual di_status allreduce_f64(double *dev, int count, cudaStream_t st) = 0;
  virtual di_status allreduce_i64(int64_t *dev, int count, cudaStream_t st) = 0;
  virtual di_status allreduce_u32(uint32_t *dev, int64_t count, cudaStream_t st) = 0;
  // every rank's `bytes` from `send` into recv[rank * bytes ...] on every rank
  virtual di_status allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;
  // grouped point-to-point: to every peer p != rank send sbytes[p] bytes from sbuf[p] and receive
  // rbytes[p] bytes into rbuf[p] (sizes agreed beforehand; 0 = nothing). Enqueued on st.
  virtual di_status exchange(const void *const *sbuf, const size_t *sbytes, void *const *rbuf,
                             const size_t *rbytes, cudaStream_t st) = 0;
  // dense fallback of the exchange: owner p receives recv[k] = sum over ranks of
  // send[b[p] + k], k < b[p+1] - b[p] (send: every rank's global-size accumulator; recv: this
  // rank's slice). Enqueued on st; send may be modified once the call returns (stream order).
  virtual di_status reduce_segments(const double *send, double *recv, const int64_t *b,
                                    cudaStream_t st) = 0;
  // Peer-memory inbox (collective; the same `bytes` on every rank): allocates this rank's
  // inbox and returns, for every rank p, a pointer to p's inbox that THIS rank's kernels can
  // store to (peers[rank] = the local inbox). NCCL: ncclMemAlloc + a symmetric window
  // (ncclCommWindowRegister) and its LSA peer pointers (NVLink P2P mappings); group: plain
  // device pointers of one GPU. DI_ENCCL when the window cannot be created (the caller then
  // moves the lists with exchange()).
  virtual di_status make_inbox(size_t bytes, std::vector<char *> *peers) = 0;
  virtual void free_inbox() = 0;
};

// In-process rank group (di_group): a generation barrier plus per-rank mailboxes.
struct Group {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<double>> red_f;    // allreduce staging, one host vector per rank
  std::vector<std::vector<int64_t>> red_i;
  std::vector<std::vector<uint32_t>> red_u;
  std::vector<std::vector<char>> gat;        // allgather staging
  std::vector<std::vector<const void *>> sptr;  // sptr[src][dst]
  std::vector<std::vector<size_t>> sbytes;
  std::vector<const double *> dsend;         // reduce_segments: every rank's accumulator
  std::vector<char *> inbox;                 // make_inbox: every rank's inbox
  int handles = 0;                           // graphs built on this group (for di_group_free)
  bool aborted = false;                      // di_group_abort: every barrier fails from now on
  explicit Group(int w)
      : world(w), red_f(w), red_i(w), red_u(w), gat(w), sptr(w, std::vector<const void *>(w, nullptr)),
        sbytes(w, std::vector<size_t>(w, 0)), dsend(w, nullptr),
        inbox(w, nullptr) {}
  // false once the group is aborted (a rank failed: the others must not wait for it forever)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) return false;
    const uint64_t my = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my || aborted; });
    }
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

// factories (comm.cu); *out = nullptr on failure, message in di_last_error
di_status make_nccl_comm(const void *unique_id, int rank, int world, Comm **out);
di_status make_group_comm(Group *grp, int rank, Comm **out);
di_status nccl_unique_id(void *out128);

}  // namespace di
