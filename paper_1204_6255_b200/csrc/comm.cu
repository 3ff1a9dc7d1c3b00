// comm.cu — NCCL (dlopen'ed) and in-process group backends of the Comm interface (comm.cuh).
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "comm.cuh"

namespace di {
namespace {

// ------------------------------------------------------------------ NCCL entry points
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  // symmetric memory (optional: the peer-memory inbox)
  ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
  ncclResult_t (*MemFree)(void *) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};

const NcclApi &nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the copy torch loaded (RTLD_NOLOAD), else whatever the loader finds
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return a;
    }
#define DI_SYM(f)                                                          \
  a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f));              \
  if (!a.f) {                                                              \
    a.why = "libnccl.so.2 lacks nccl" #f;                                  \
    return a;                                                              \
  }
    DI_SYM(GetUniqueId)
    DI_SYM(CommInitRank)
    DI_SYM(CommDestroy)
    DI_SYM(AllReduce)
    DI_SYM(AllGather)
    DI_SYM(Reduce)
    DI_SYM(Send)
    DI_SYM(Recv)
    DI_SYM(GroupStart)
    DI_SYM(GroupEnd)
    DI_SYM(GetErrorString)
#undef DI_SYM
    a.MemAlloc = reinterpret_cast<decltype(a.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
    a.MemFree = reinterpret_cast<decltype(a.MemFree)>(dlsym(h, "ncclMemFree"));
    a.CommWindowRegister =
        reinterpret_cast<decltype(a.CommWindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
    a.CommWindowDeregister =
        reinterpret_cast<decltype(a.CommWindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
    a.ok = true;
    return a;
  }();
  return api;
}

#define DI_NCK(call)                                                                    \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      ::di::set_error(std::string(#call) + ": " + nccl().GetErrorString(r_));           \
      return DI_ENCCL;                                                                  \
    }                                                                                   \
  } while (0)

// the LSA (NVLink load/store) pointers of every rank's window, read on the device
__global__ void k_window_peers(ncclWindow_t w, int world, char **out) {
  for (int p = threadIdx.x; p < world; p += blockDim.x)
    out[p] = static_cast<char *>(ncclGetPeerPointer(w, 0, p));
}

// Communicators by unique id: an ncclUniqueId initialises exactly one communicator (a second
// ncclCommInitRank with the same id is not supported), so every graph uploaded with the same
// (id, rank, world) shares one, e.g. the e2e uploads of bench.py at N > 1. They live until the
// process exits and are never destroyed (NCCL may already be unloaded at static destruction).
// The map's mutex is held only to find / insert an entry; the collective ncclCommInitRank runs
// outside it, once per entry (std::call_once), so ranks driven by threads of one process do not
// wait for each other's initialisation behind the mutex.
struct CommEntry {
  std::once_flag once;
  ncclComm_t comm = nullptr;
  ncclResult_t res = ncclSuccess;
};
std::mutex g_comm_mu;
std::map<std::string, std::shared_ptr<CommEntry>> *g_comms =
    new std::map<std::string, std::shared_ptr<CommEntry>>();

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;   // shared (g_comms), not owned
  void *ibuf = nullptr;
  ncclWindow_t iwin = nullptr;
  ~NcclComm() override { free_inbox(); }
  di_status make_inbox(size_t bytes, std::vector<char *> *peers) override {
    const NcclApi &a = nccl();
    if (!a.MemAlloc || !a.MemFree || !a.CommWindowRegister || !a.CommWindowDeregister) {
      set_error("libnccl.so.2 lacks the symmetric-memory API (ncclMemAlloc / ncclCommWindowRegister)");
      return DI_ENCCL;
    }
    free_inbox();
    bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT *
            NCCL_WIN_REQUIRED_ALIGNMENT;
    DI_NCK(a.MemAlloc(&ibuf, bytes));
    ncclResult_t r = a.CommWindowRegister(comm, ibuf, bytes, &iwin, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
      set_error(std::string("ncclCommWindowRegister: ") + a.GetErrorString(r));
      a.MemFree(ibuf);
      ibuf = nullptr;
      iwin = nullptr;
      return DI_ENCCL;
    }
    char **dp = nullptr;
    DI_CK(cudaMalloc(&dp, sizeof(char *) * world));
    k_window_peers<<<1, 32>>>(iwin, world, dp);
    peers->assign(world, nullptr);
    cudaError_t e = cudaMemcpy(peers->data(), dp, sizeof(char *) * world, cudaMemcpyDeviceToHost);
    cudaFree(dp);
    DI_CK(e);
    return DI_OK;
  }
  void free_inbox() override {
    if (iwin) nccl().CommWindowDeregister(comm, iwin);
    if (ibuf) nccl().MemFree(ibuf);
    iwin = nullptr;
    ibuf = nullptr;
  }
  di_status allreduce_f64(double *dev, int count, cudaStream_t st) override {
    DI_NCK(nccl().AllReduce(dev, dev, (size_t)count, ncclFloat64, ncclSum, comm, st));
    return DI_OK;
  }
  di_status allreduce_i64(int64_t *dev, int count, cudaStream_t st) override {
    DI_NCK(nccl().AllReduce(dev, dev, (size_t)count, ncclInt64, ncclSum, comm, st));
    return DI_OK;
  }
  di_status allreduce_u32(uint32_t *dev, int64_t count, cudaStream_t st) override {
    DI_NCK(nccl().AllReduce(dev, dev, (size_t)count, ncclUint32, ncclSum, comm, st));
    return DI_OK;
  }
  di_status allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    DI_NCK(nccl().AllGather(send, recv, bytes, ncclUint8, comm, st));
    return DI_OK;
  }
  di_status exchange(const void *const *sbuf, const size_t *sbytes, void *const *rbuf,
                     const size_t *rbytes, cudaStream_t st) override {
    DI_NCK(nccl().GroupStart());
    for (int p = 0; p < world; p++) {
      if (p == rank) continue;
      if (sbytes[p]) DI_NCK(nccl().Send(sbuf[p], sbytes[p], ncclUint8, p, comm, st));
      if (rbytes[p]) DI_NCK(nccl().Recv(rbuf[p], rbytes[p], ncclUint8, p, comm, st));
    }
    DI_NCK(nccl().GroupEnd());
    return DI_OK;
  }
  di_status reduce_segments(const double *send, double *recv, const int64_t *b,
                            cudaStream_t st) override {
    DI_NCK(nccl().GroupStart());   // one reduction per owner (ranges differ in size)
    for (int p = 0; p < world; p++)
      DI_NCK(nccl().Reduce(send + b[p], recv, (size_t)(b[p + 1] - b[p]), ncclFloat64, ncclSum, p,
                           comm, st));
    DI_NCK(nccl().GroupEnd());
    return DI_OK;
  }
};

// group backend's dense reduction: this rank's slice summed over every rank's accumulator, in
// rank order (the values are the same on every run)
struct SendPtrs {
  const double *p[kMaxWorld];
};
__global__ void k_sum_segments(SendPtrs sp, int world, int64_t off, int64_t n, double *recv) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < world; q++) s += sp.p[q][off + k];
    recv[k] = s;
  }
}

// ------------------------------------------------------------------ in-process group
struct GroupComm : Comm {
  Group *g = nullptr;
  di_status aborted() {
    set_error("in-process group aborted (another rank failed)");
    return DI_ESTATE;
  }
  template <typename T>
  di_status allreduce(T *dev, int64_t count, cudaStream_t st, std::vector<std::vector<T>> &stage) {
    std::vector<T> &mine = stage[rank];
    mine.assign((size_t)count, T(0));
    DI_CK(cudaMemcpyAsync(mine.data(), dev, (size_t)count * sizeof(T), cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    if (!g->barrier()) return aborted();
    std::vector<T> sum((size_t)count, T(0));
    for (int p = 0; p < world; p++)  // rank order: every rank computes the identical sum
      for (int64_t k = 0; k < count; k++) sum[k] += stage[p][k];
    if (!g->barrier()) return aborted();  // nobody restages before everyone has summed
    DI_CK(cudaMemcpyAsync(dev, sum.data(), (size_t)count * sizeof(T), cudaMemcpyHostToDevice, st));
    DI_CK(cudaStreamSynchronize(st));
    return DI_OK;
  }
  di_status allreduce_f64(double *dev, int count, cudaStream_t st) override {
    return allreduce(dev, count, st, g->red_f);
  }
  di_status allreduce_i64(int64_t *dev, int count, cudaStream_t st) override {
    return allreduce(dev, count, st, g->red_i);
  }
  di_status allreduce_u32(uint32_t *dev, int64_t count, cudaStream_t st) override {
    return allreduce(dev, count, st, g->red_u);
  }
  di_status allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
    std::vector<char> &mine = g->gat[rank];
    mine.resize(bytes);
    DI_CK(cudaMemcpyAsync(mine.data(), send, bytes, cudaMemcpyDeviceToHost, st));
    DI_CK(cudaStreamSynchronize(st));
    if (!g->barrier()) return aborted();
    for (int p = 0; p < world; p++)
      DI_CK(cudaMemcpyAsync((char *)recv + (size_t)p * bytes, g->gat[p].data(), bytes,
                            cudaMemcpyHostToDevice, st));
    DI_CK(cudaStreamSynchronize(st));
    if (!g->barrier()) return aborted();  // nobody restages before everyone has copied
    return DI_OK;
  }
  di_status exchange(const void *const *sbuf, const size_t *sbytes, void *const *rbuf,
                     const size_t *rbytes, cudaStream_t st) override {
    DI_CK(cudaStreamSynchronize(st));  // send buffers complete
    for (int p = 0; p < world; p++) {
      g->sptr[rank][p] = (p == rank) ? nullptr : sbuf[p];
      g->sbytes[rank][p] = (p == rank) ? 0 : sbytes[p];
    }
    if (!g->barrier()) return aborted();
    di_status s = DI_OK;
    for (int p = 0; p < world; p++) {
      if (p == rank) continue;
      if (g->sbytes[p][rank] != rbytes[p]) {
        set_error("group exchange: rank " + std::to_string(p) + " sends " +
                  std::to_string(g->sbytes[p][rank]) + " bytes to rank " + std::to_string(rank) +
                  ", which expects " + std::to_string(rbytes[p]));
        s = DI_ESTATE;
        continue;
      }
      if (rbytes[p] &&
          cudaMemcpyAsync(rbuf[p], g->sptr[p][rank], rbytes[p], cudaMemcpyDeviceToDevice, st) !=
              cudaSuccess)
        s = DI_ECUDA;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && s == DI_OK) s = DI_ECUDA;
    // senders may reuse their buffers only after every receiver copied
    if (!g->barrier()) return aborted();
    if (s != DI_OK) g->abort();
    return s;
  }
  char *ibuf = nullptr;
  ~GroupComm() override { free_inbox(); }
  di_status make_inbox(size_t bytes, std::vector<char *> *peers) override {
    free_inbox();
    DI_CK(cudaMalloc(&ibuf, bytes));
    g->inbox[rank] = ibuf;
    if (!g->barrier()) return aborted();
    peers->assign(g->inbox.begin(), g->inbox.end());
    if (!g->barrier()) return aborted();
    return DI_OK;
  }
  void free_inbox() override {
    if (ibuf) cudaFree(ibuf);
    ibuf = nullptr;
  }
  di_status reduce_segments(const double *send, double *recv, const int64_t *b,
                            cudaStream_t st) override {
    DI_CK(cudaStreamSynchronize(st));  // this rank's accumulator complete
    g->dsend[rank] = send;
    if (!g->barrier()) return aborted();
    SendPtrs sp{};
    for (int q = 0; q < world; q++) sp.p[q] = g->dsend[q];
    const int64_t n = b[rank + 1] - b[rank];
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184));
    k_sum_segments<<<grid, 256, 0, st>>>(sp, world, b[rank], n, recv);
    di_status s = (cudaGetLastError() == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess)
                      ? DI_OK
                      : DI_ECUDA;
    // owners may clear their accumulators only after every rank has read them
    if (!g->barrier()) return aborted();
    if (s != DI_OK) g->abort();
    return s;
  }
};

}  // namespace

di_status nccl_unique_id(void *out128) {
  const NcclApi &a = nccl();
  if (!a.ok) {
    set_error(a.why);
    return DI_ENCCL;
  }
  ncclUniqueId id;
  DI_NCK(a.GetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return DI_OK;
}

di_status make_nccl_comm(const void *unique_id, int rank, int world, Comm **out) {
  *out = nullptr;
  const NcclApi &a = nccl();
  if (!a.ok) {
    set_error(a.why);
    return DI_ENCCL;
  }
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  std::string key(reinterpret_cast<const char *>(&id), sizeof(id));
  key += ":" + std::to_string(rank) + "/" + std::to_string(world);
  std::shared_ptr<CommEntry> e;
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    std::shared_ptr<CommEntry> &slot = (*g_comms)[key];
    if (!slot) slot = std::make_shared<CommEntry>();
    e = slot;
  }
  std::call_once(e->once, [&] { e->res = a.CommInitRank(&e->comm, world, id, rank); });
  if (e->res != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + a.GetErrorString(e->res));
    return DI_ENCCL;
  }
  ncclComm_t comm = e->comm;
  NcclComm *c = new NcclComm();
  c->rank = rank;
  c->world = world;
  c->comm = comm;
  *out = c;
  return DI_OK;
}

di_status make_group_comm(Group *grp, int rank, Comm **out) {
  GroupComm *c = new GroupComm();
  c->g = grp;
  c->rank = rank;
  c->world = grp->world;
  *out = c;
  return DI_OK;
}

}  // namespace di
