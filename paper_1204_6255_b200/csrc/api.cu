// api.cu — C ABI of libdi.so (include/di.h, include/di_test.h): handle management and the
// host side of the sweep loop. The loop enqueues sweeps in batches without reading anything
// back in between; the device finaliser decides convergence and later
// kernels no-op, so the host only synchronises once per batch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/di.h"
#include "../../include/di_test.h"
#include "comm.cuh"
#include "di_common.cuh"

namespace di {

static std::mutex g_opt_mu;
static Options g_opt;
Options options() {
  std::lock_guard<std::mutex> lk(g_opt_mu);
  return g_opt;
}

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

cudaStream_t &alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

cudaError_t dmalloc_bytes(void **p, size_t bytes) {
  static thread_local int prepared = -1;  // device whose pool was configured by this thread
  int dev = 0;
  cudaGetDevice(&dev);
  if (prepared != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;  // keep freed memory in the pool for the next upload / solve
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    prepared = dev;
  }
  const bool trace = options().build_trace != 0;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 1, alloc_stream());
  // the buffer is then usable on any stream (some host paths touch it with synchronous copies)
  if (e == cudaSuccess) e = cudaStreamSynchronize(alloc_stream());
  if (trace && bytes >= (64u << 20))
    fprintf(stderr, "[di alloc] %8.1f MB %8.2f ms\n", bytes / 1e6,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  return e;
}

// Pinned host mirrors of the per-graph Scalars from a process-wide slab (cudaMallocHost /
// cudaFreeHost per upload cost ms and cudaFreeHost synchronises the device): slabs of 64 mirrors,
// never returned to the driver, handed out and back under a mutex.
static std::mutex g_pin_mu;
static std::vector<Scalars *> g_pin_free;
cudaError_t pinned_scalars_get(Scalars **out) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  if (g_pin_free.empty()) {
    Scalars *slab = nullptr;
    cudaError_t e = cudaMallocHost(&slab, 64 * sizeof(Scalars));
    if (e != cudaSuccess) return e;
    for (int k = 63; k >= 0; k--) g_pin_free.push_back(slab + k);
  }
  *out = g_pin_free.back();
  g_pin_free.pop_back();
  return cudaSuccess;
}
void pinned_scalars_put(Scalars *p) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(p);
}

void dfree(void *p) {
  if (p) cudaFreeAsync(p, alloc_stream());
}

cudaError_t dmemset(void *p, int v, size_t bytes) {
  return cudaMemsetAsync(p, v, bytes, alloc_stream());
}

namespace {

__global__ void k_check_B(const double *B, int64_t n, int *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double b = B[i];
    if (!(b >= 0.0) || !isfinite(b)) *bad = 1;
  }
}

// out[k] = in[idx[k]] (idx = NULL: plain copy)
__global__ void k_gather(double *__restrict__ out, const double *__restrict__ in,
                         const int32_t *__restrict__ idx, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[idx ? idx[k] : k];
}

void gather(const Graph &g, double *out, const double *in, const int32_t *idx) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((g.n + 255) / 256, 16 * g.num_sms));
  k_gather<<<grid, 256, 0, g.stream>>>(out, in, idx, g.n);
}

di_status fail(di_status s, const std::string &msg) {
  set_error(msg);
  return s;
}

struct EventSet {
  std::vector<cudaEvent_t> ev;
  ~EventSet() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaEvent_t get(size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[i];
  }
};

void free_graph(Graph *g) {
  if (!g) return;
  void *ptrs[] = {g->cold_rec, g->cold_off, g->cold_top, g->cold_fill, g->ppartials, g->rep, g->hub_items, g->cyc_times, g->row_ptr, g->col, g->deg, g->kloop, g->csc_ptr, g->csc_row, g->F, g->H,
                  g->new_of, g->old_of, g->Bperm, g->xfer,
                  g->S, g->aux, g->sc, g->partials, g->ipartials, g->red_partials,
                  g->log_r, g->log_sel, g->log_links, g->log_mode};
  for (void *p : ptrs)
    if (p) dfree(p);
  for (int b = 0; b < kBins; b++) {
    void *q[] = {g->fr.ent[b], g->fr.id[b]};
    for (void *p : q)
      if (p) dfree(p);
  }
  for (int b = 0; b < kPullBins; b++) {
    if (g->pe[b]) dfree(g->pe[b]);
    if (g->re[b]) dfree(g->re[b]);
  }
  if (g->cmp_partials) dfree(g->cmp_partials);
  if (g->loop_exec) cudaGraphExecDestroy(g->loop_exec);
  if (g->loop_graph) cudaGraphDestroy(g->loop_graph);
  if (g->sc_host) pinned_scalars_put(g->sc_host);
  free_dist(*g);
  if (g->group) {
    std::lock_guard<std::mutex> lk(g->group->m);
    g->group->handles--;
  }
  delete g;
}

// The sweep loop as one CUDA graph: a while node whose body is one cycle (blocks x (select,
// push|pull)) followed by k_loop_cond, which keeps looping while !stop && sweeps < max_sweeps.
// The host launches it once and synchronises once (plus the exact residual check).
di_status loop_graph(Graph &g, int blocks, int mode, bool async) {
  const int key = (blocks * 4 + mode) * 2 + (async ? 1 : 0);
  if (g.loop_exec && g.loop_key == key) return DI_OK;
  if (g.loop_exec) cudaGraphExecDestroy(g.loop_exec);
  if (g.loop_graph) cudaGraphDestroy(g.loop_graph);
  g.loop_exec = nullptr;
  g.loop_graph = nullptr;
  cudaGraph_t gr;
  DI_CK(cudaGraphCreate(&gr, 0));
  cudaGraphConditionalHandle h;
  DI_CK(cudaGraphConditionalHandleCreate(&h, gr, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  DI_CK(cudaGraphAddNode(&node, gr, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  // capture on a private stream (the handle's stream may be the legacy default stream, which
  // cannot capture); the graph is launched on the handle's stream
  cudaStream_t user = g.stream, cs = nullptr;
  DI_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  g.stream = cs;
  cudaError_t be = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeThreadLocal);
  if (be != cudaSuccess) {
    g.stream = user;
    cudaStreamDestroy(cs);
    cudaGraphDestroy(gr);
    return fail(DI_ECUDA, std::string("DI_GRAPH_LOOP capture: ") + cudaGetErrorString(be));
  }
  int64_t launches = 0;
  for (int b = 0; b < blocks; b++) {
    if (async) {
      launch_cycle(g, &launches);
      continue;
    }
    launch_select(g, 0, &launches, b, blocks);
    if (mode != MODE_PULL) launch_push(g, &launches, b, blocks);
    if (mode != MODE_PUSH) launch_pull(g, &launches);
  }
  launch_loop_cond(g, h);
  launches++;
  cudaGraph_t cap = body;
  cudaError_t ce = cudaStreamEndCapture(cs, &cap);
  g.stream = user;
  cudaStreamDestroy(cs);
  if (ce != cudaSuccess) {
    cudaGraphDestroy(gr);
    return fail(DI_ECUDA, std::string("DI_GRAPH_LOOP capture: ") + cudaGetErrorString(ce));
  }
  ce = cudaGraphInstantiate(&g.loop_exec, gr, 0);
  if (ce != cudaSuccess) {
    cudaGraphDestroy(gr);
    g.loop_exec = nullptr;
    return fail(DI_ECUDA, std::string("DI_GRAPH_LOOP instantiate: ") + cudaGetErrorString(ce));
  }
  g.loop_graph = gr;
  g.loop_key = key;
  g.loop_launches = launches;
  return DI_OK;
}

di_status sync_scalars(Graph &g) {
  DI_CK(cudaMemcpyAsync(g.sc_host, g.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, g.stream));
  DI_CK(cudaStreamSynchronize(g.stream));
  return DI_OK;
}

}  // namespace
}  // namespace di

using namespace di;

extern "C" {

const char *di_last_error(void) { return g_err.c_str(); }

di_status di_nccl_unique_id(void *out128) {
  if (!out128) return fail(DI_EINVAL, "di_nccl_unique_id: NULL argument");
  return nccl_unique_id(out128);
}

di_status di_group_create(int32_t world, di_group *out) {
  if (!out) return fail(DI_EINVAL, "di_group_create: NULL argument");
  *out = nullptr;
  if (world < 1 || world > kMaxWorld)
    return fail(DI_EINVAL, "di_group_create: world must be in [1, " + std::to_string(kMaxWorld) + "]");
  *out = (di_group) new Group(world);
  return DI_OK;
}

di_status di_group_abort(di_group grp) {
  Group *g = (Group *)grp;
  if (!g) return fail(DI_EINVAL, "di_group_abort: NULL group");
  g->abort();
  return DI_OK;
}

di_status di_group_free(di_group grp) {
  Group *g = (Group *)grp;
  if (!g) return DI_OK;
  {
    std::lock_guard<std::mutex> lk(g->m);
    if (g->handles > 0) return fail(DI_ESTATE, "di_group_free: graphs of this group are still alive");
  }
  delete g;
  return DI_OK;
}

di_status di_graph_upload(const int32_t *src, const int32_t *dst, int64_t n_links, int64_t n_nodes,
                          uint32_t flags, void *stream, const di_dist *dist, di_graph *out) {
  if (!out) return fail(DI_EINVAL, "di_graph_upload: out is NULL");
  *out = nullptr;
  if (n_nodes < 1 || n_nodes > 2147483647LL)
    return fail(DI_EINVAL, "di_graph_upload: n_nodes must be in [1, 2^31-1]");
  if (n_links < 0) return fail(DI_EINVAL, "di_graph_upload: n_links < 0");
  if (n_links > 0 && (!src || !dst)) return fail(DI_EINVAL, "di_graph_upload: NULL src/dst");
  const int world = dist ? dist->world : 1;
  Group *grp = dist ? (Group *)dist->group : nullptr;
  const int rank = dist ? dist->rank : 0;
  if (world < 1 || world > kMaxWorld)
    return fail(DI_EINVAL, "di_graph_upload: dist->world must be in [1, " +
                               std::to_string(kMaxWorld) + "]");
  if (rank < 0 || rank >= world) return fail(DI_EINVAL, "di_graph_upload: dist->rank out of range");
  // partitioned: any rank of a communicator, including a communicator of one rank (which runs
  // the whole multi-GPU protocol with nothing to exchange: tests the NCCL backend on one GPU)
  const bool partitioned = dist && (world > 1 || grp || dist->nccl_unique_id);
  if (!partitioned && (flags & DI_LOCAL_LINKS))
    return fail(DI_EINVAL, "di_graph_upload: DI_LOCAL_LINKS is for partitioned graphs");
  if (partitioned) {
    if (n_nodes < world) return fail(DI_EINVAL, "di_graph_upload: fewer nodes than ranks");
    if (flags & DI_BUILD_CSC)
      return fail(DI_EINVAL, "di_graph_upload: DI_BUILD_CSC is single-GPU (partitioned sweeps are "
                             "push-only)");
    // (a DI_LOCAL_LINKS range outside [0, n) is reported by the collective validation in
    //  build_graph, on every rank: a rank must not leave before the communicator exists)
    if (!grp && !dist->nccl_unique_id)
      return fail(DI_EINVAL, "di_graph_upload: dist needs an NCCL unique id or a di_group");
    if (grp && grp->world != world)
      return fail(DI_EINVAL, "di_graph_upload: dist->world differs from the group's size");
  }
  int dev = 0, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(DI_ECUDA, "di_graph_upload: no CUDA device");
  DI_CK(cudaGetDevice(&dev));
  AllocScope as((cudaStream_t)stream);
  Graph *g = new Graph();
  g->device = dev;
  g->stream = (cudaStream_t)stream;
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, dev);
  g->n = g->n_global = n_nodes;
  g->lo = 0;
  g->hi = n_nodes;
  g->rank = rank;
  g->world = world;
  g->partitioned = partitioned;
  if (partitioned) {  // the communicator first: ncclCommInitRank is collective
    Comm *c = nullptr;
    di_status cs = grp ? make_group_comm(grp, rank, &c)
                       : make_nccl_comm(dist->nccl_unique_id, rank, world, &c);
    if (cs != DI_OK) {
      delete g;
      return cs;
    }
    g->comm = c;
    if (grp) {
      g->group = grp;
      std::lock_guard<std::mutex> lk(g->group->m);
      g->group->handles++;
    }
  }
  if (partitioned && (flags & DI_LOCAL_LINKS)) {
    g->local_links = true;
    g->local_lo = dist->lo;
    g->local_hi = dist->hi;
  }
  {
    const Options o = options();
    g->red_hint = o.red_hint;
    g->push_occ = o.push_occ;
    g->auto_ratio = o.auto_ratio;
    g->stripes = o.stripes;
    g->hot_acc = o.hot_acc;
    g->repl_share = o.repl_share;
    g->cold_mode = o.cold_bins;
    g->cold_tier = o.cold_tier;
    g->grid_div = o.cycle_grid_div;
    g->cycle_times = o.cycle_times;
    g->p2p_opt = o.p2p;
    g->p2p_force = o.p2p_force;
    g->remote_compact = o.remote_compact;
    g->remote_tier = o.remote_tier;
    g->long_lanes = o.long_lanes;
    g->row_sort = o.row_sort;
    g->line_spread = o.line_spread;
    g->cold_shift_opt = o.cold_shift;
    g->warm_opt = o.warm;
    g->warm_flush = o.warm_flush;
    g->warm_shift_opt = o.warm_shift;
    g->dist_parts = o.dist_parts;
  }
  di_status s = build_graph(*g, src, dst, n_links, flags);
  btrace("built");
  if (s == DI_OK) s = alloc_state(*g);
  btrace("state");
  if (s == DI_OK) s = alloc_pull(*g);
  btrace("pull");
  if (s == DI_OK && partitioned) s = alloc_dist(*g);
  if (s != DI_OK) {
    free_graph(g);
    return s;
  }
  *out = (di_graph)g;
  return DI_OK;
}

namespace {
struct OptDesc {
  const char *name;
  double lo, hi;
  bool integer;
};
const OptDesc kOpts[] = {
    {"red_hint", 0, 1, true},       {"push_occ", 1, 32, true},    {"auto_ratio", 0, 1e9, false},
    {"stripes", 0, 2147483647.0, true}, {"hot_acc", 0, 1, true},  {"repl_share", 0, 1, false},
    {"cold_bins", -1, 1, true},     {"cold_tier", 0, 2147483647.0, true},
    {"cycle_grid_div", 1, 4096, true}, {"cycle_times", 0, 1, true}, {"p2p", 0, 1, true},
    {"p2p_force", 0, 1, true},      {"build_trace", 0, 1, true},
    {"remote_compact", 0, 1, true}, {"remote_tier", 0, 2147483647.0, true},
    {"long_lanes", 0, 1, true},     {"row_sort", 0, 1, true},      {"line_spread", 1, 16, true},
    {"cold_shift", 0, 30, true},     {"warm", -1, 65536, true},      {"warm_flush", 0, 1 << 20, true},
    {"warm_shift", 0, 30, true},     {"dist_parts", 1, 64, true},
};
}  // namespace

di_status di_set_option(const char *name, double value) {
  if (!name) return fail(DI_EINVAL, "di_set_option: NULL name");
  const std::string n(name);
  const OptDesc *d = nullptr;
  for (const auto &k : kOpts)
    if (n == k.name) d = &k;
  if (!d) return fail(DI_EINVAL, "di_set_option: unknown option '" + n + "'");
  if (!std::isfinite(value) || value < d->lo || value > d->hi || (d->integer && value != std::floor(value)))
    return fail(DI_EINVAL, "di_set_option: value out of range for '" + n + "'");
  std::lock_guard<std::mutex> lk(g_opt_mu);
  Options &o = g_opt;
  const int iv = (int)value;
  if (n == "red_hint") o.red_hint = iv;
  else if (n == "push_occ") o.push_occ = iv;
  else if (n == "auto_ratio") o.auto_ratio = value;
  else if (n == "stripes") o.stripes = iv;
  else if (n == "hot_acc") o.hot_acc = iv;
  else if (n == "repl_share") o.repl_share = value;
  else if (n == "cold_bins") o.cold_bins = iv;
  else if (n == "cold_tier") o.cold_tier = (int64_t)value;
  else if (n == "cycle_grid_div") o.cycle_grid_div = iv;
  else if (n == "cycle_times") o.cycle_times = iv;
  else if (n == "p2p") o.p2p = iv;
  else if (n == "p2p_force") o.p2p_force = iv;
  else if (n == "build_trace") o.build_trace = iv;
  else if (n == "remote_compact") o.remote_compact = iv;
  else if (n == "remote_tier") o.remote_tier = (int64_t)value;
  else if (n == "long_lanes") o.long_lanes = iv;
  else if (n == "row_sort") o.row_sort = iv;
  else if (n == "cold_shift") o.cold_shift = iv;
  else if (n == "warm") o.warm = iv;
  else if (n == "warm_flush") o.warm_flush = iv;
  else if (n == "warm_shift") o.warm_shift = iv;
  else if (n == "dist_parts") o.dist_parts = iv;
  else if (n == "line_spread") {
    if (iv != 1 && iv != 2 && iv != 4 && iv != 8 && iv != 16)
      return fail(DI_EINVAL, "di_set_option: line_spread must be 1, 2, 4, 8 or 16");
    o.line_spread = iv;
  }
  return DI_OK;
}

di_status di_get_option(const char *name, double *value) {
  if (!name || !value) return fail(DI_EINVAL, "di_get_option: NULL argument");
  const std::string n(name);
  const Options o = options();
  if (n == "red_hint") *value = o.red_hint;
  else if (n == "push_occ") *value = o.push_occ;
  else if (n == "auto_ratio") *value = o.auto_ratio;
  else if (n == "stripes") *value = o.stripes;
  else if (n == "hot_acc") *value = o.hot_acc;
  else if (n == "repl_share") *value = o.repl_share;
  else if (n == "cold_bins") *value = o.cold_bins;
  else if (n == "cold_tier") *value = (double)o.cold_tier;
  else if (n == "cycle_grid_div") *value = o.cycle_grid_div;
  else if (n == "cycle_times") *value = o.cycle_times;
  else if (n == "p2p") *value = o.p2p;
  else if (n == "p2p_force") *value = o.p2p_force;
  else if (n == "build_trace") *value = o.build_trace;
  else if (n == "remote_compact") *value = o.remote_compact;
  else if (n == "remote_tier") *value = (double)o.remote_tier;
  else if (n == "long_lanes") *value = o.long_lanes;
  else if (n == "row_sort") *value = o.row_sort;
  else if (n == "warm") *value = o.warm;
  else if (n == "warm_flush") *value = o.warm_flush;
  else if (n == "warm_shift") *value = o.warm_shift;
  else if (n == "dist_parts") *value = o.dist_parts;
  else if (n == "line_spread") *value = o.line_spread;
  else if (n == "cold_shift") *value = o.cold_shift;
  else return fail(DI_EINVAL, "di_get_option: unknown option '" + n + "'");
  return DI_OK;
}

di_status di_set_threshold_scale(di_graph h, double alpha) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "di_set_threshold_scale: NULL handle");
  if (!(alpha > 0.0) || !std::isfinite(alpha))
    return fail(DI_EINVAL, "di_set_threshold_scale: alpha must be finite and > 0");
  g->alpha = alpha;
  return DI_OK;
}

di_status di_graph_set_stream(di_graph h, void *stream) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "di_graph_set_stream: NULL handle");
  DI_CK(cudaStreamSynchronize(g->stream));   // the old stream's work is done before the switch
  g->stream = (cudaStream_t)stream;
  return DI_OK;
}

di_status di_graph_range(di_graph h, int64_t *lo, int64_t *hi) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "NULL handle");
  if (lo) *lo = g->lo;
  if (hi) *hi = g->hi;
  return DI_OK;
}

di_status di_graph_links(di_graph h, int64_t *n_links) {
  Graph *g = (Graph *)h;
  if (!g || !n_links) return fail(DI_EINVAL, "NULL argument");
  *n_links = g->l;
  return DI_OK;
}

di_status di_graph_free(di_graph h) {
  Graph *g = (Graph *)h;
  if (!g) return DI_OK;
  AllocScope as(g->stream);
  cudaStreamSynchronize(g->stream);
  cudaStream_t st = g->stream;
  free_graph(g);
  cudaStreamSynchronize(st);
  return DI_OK;
}

di_status di_solve(di_graph h, double d, const double *B, double tol, di_variant v,
                   int64_t max_sweeps, uint32_t flags, di_stats *st) {
  Graph *gp = (Graph *)h;
  if (!gp) return fail(DI_EINVAL, "di_solve: NULL handle");
  Graph &g = *gp;
  AllocScope as(g.stream);
  if (!(d > 0.0 && d < 1.0)) return fail(DI_EINVAL, "di_solve: d must be in (0, 1)");
  if (!(tol > 0.0) || !std::isfinite(tol)) return fail(DI_EINVAL, "di_solve: tol must be > 0");
  if (max_sweeps < 0) return fail(DI_EINVAL, "di_solve: max_sweeps < 0");
  if ((int)v < 0 || (int)v > DI_GS_BLOCK) return fail(DI_EINVAL, "di_solve: bad variant");
  if (B) {
    int *bad = nullptr;
    DI_CK(dmalloc(&bad, 4));
    DI_CK(cudaMemsetAsync(bad, 0, 4, g.stream));
    k_check_B<<<std::max<int64_t>(1, std::min<int64_t>((g.n + 255) / 256, 4096)), 256, 0,
                g.stream>>>(B, g.n, bad);
    int hb = 0;
    DI_CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, g.stream));
    DI_CK(cudaStreamSynchronize(g.stream));
    dfree(bad);
    if (hb) return fail(DI_EINVAL, "di_solve: B has a negative or non-finite entry");
  }
  if (g.partitioned) {
    if (v != DI_SOP && v != DI_CYC)
      return fail(DI_EINVAL, "di_solve: a partitioned graph runs DI_SOP / DI_CYC only");
    if ((flags & (DI_PULL | DI_AUTO | DI_GRAPH_LOOP)) || ((flags >> 16) & 0xFFu) > 1)
      return fail(DI_EINVAL, "di_solve: a partitioned graph runs push sweeps (bulk or DI_ASYNC)");
    if ((flags & DI_RESUME) && !g.solved) return fail(DI_ESTATE, "di_solve: DI_RESUME before any solve");
    const double *Bint = B;
    if (B && g.reordered) {  // caller's slice [lo, hi) in the caller's numbering
      if (!g.Bperm) DI_CK(dmalloc(&g.Bperm, (size_t)g.n * 8));
      gather(g, g.Bperm, B - g.lo, g.old_of + g.lo);
      Bint = g.Bperm;
    }
    return solve_dist(g, d, Bint, tol, (int)v, max_sweeps, flags, st);
  }
  if (v == DI_PI_PULL || v == DI_PI_PUSH || v == DI_GS_BLOCK) {
    if (v == DI_PI_PUSH) {   // PI' push uses the replicated hot accumulators too
      di_status ps = prepare_cycle(g, false);
      if (ps != DI_OK) return ps;
    }
    return run_comparator(g, d, tol, (int)v, max_sweeps, flags, st);
  }
  const int mode = (flags & DI_PULL) ? MODE_PULL : ((flags & DI_AUTO) ? MODE_AUTO : MODE_PUSH);
  if (mode != MODE_PUSH && !g.has_csc)
    return fail(DI_EINVAL, "di_solve: DI_PULL / DI_AUTO need the CSC (upload with DI_BUILD_CSC)");
  // block-ordered cycles (F1): K sub-sweeps over ordered node blocks per cycle
  int blocks = (int)((flags >> 16) & 0xFFu);
  if (blocks < 1) blocks = 1;
  if (blocks > 1 && mode != MODE_PUSH)
    return fail(DI_EINVAL, "di_solve: block-ordered cycles (DI_BLOCKS) run push sweeps only");
  blocks = (int)std::min<int64_t>(blocks, std::max<int64_t>(1, select_tiles(g.n)));
  const bool async = flags & DI_ASYNC;
  if (async && (mode != MODE_PUSH || blocks > 1))
    return fail(DI_EINVAL, "di_solve: DI_ASYNC runs push cycles without DI_BLOCKS");
  {  // replicated hot accumulators (every push schedule) and, for DI_ASYNC, the cold bins
    di_status ps = prepare_cycle(g, async);
    if (ps != DI_OK) return ps;
  }
  const bool resume = flags & DI_RESUME;
  if (resume && !g.solved) return fail(DI_ESTATE, "di_solve: DI_RESUME before any solve");
  const int paper = (flags & DI_PAPER_ERROR) ? 1 : 0;
  const int trace = (flags & DI_TRACE) ? 1 : 0;
  const bool prof = flags & DI_PROFILE;

  int64_t launches = 0;
  cudaEvent_t t0, t1;
  DI_CK(cudaEventCreate(&t0));
  DI_CK(cudaEventCreate(&t1));
  EventSet evs;

  // fresh device scalars (the epoch keeps increasing across solves)
  {
    Scalars &s = *g.sc_host;
    const uint32_t epoch = s.epoch ? s.epoch : 1;
    const double e_prev = s.e;
    memset(&s, 0, sizeof(Scalars));
    s.epoch = epoch;
    s.e = resume ? e_prev : 0.0;
    s.d = d;
    s.tol = tol;
    s.variant = (int32_t)v;
    s.paper_err = paper;
    s.alpha = g.alpha;
    s.trace = trace;
    s.mode = mode;
    s.pull_thr = (int64_t)(g.auto_ratio * (double)g.l_global);
    s.max_sweeps = max_sweeps;
  }
  DI_CK(cudaEventRecord(t0, g.stream));
  DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  const double *Bint = B;
  if (B && g.reordered) {   // B arrives in the caller's numbering
    if (!g.Bperm) DI_CK(dmalloc(&g.Bperm, (size_t)g.n * 8));
    gather(g, g.Bperm, B, g.old_of);
    launches++;
    Bint = g.Bperm;
  }
  if (!resume)
    launch_init(g, Bint, d, &launches);
  else
    launch_reduce_F_setr(g, &launches);
  di_status s = sync_scalars(g);
  if (s != DI_OK) return s;
  auto err_of = [&](double r, double e) { return paper ? r / (1.0 - d - d * e) : r; };
  bool converged = err_of(g.sc_host->r, g.sc_host->e) <= tol;
  double resid = g.sc_host->r;
  int64_t launched = 0;
  int64_t batch = 4;
  double push_ms = 0.0, select_ms = 0.0;
  int64_t push_launches = 0;
  double r_prev = g.sc_host->r;
  const bool graph_loop = (flags & DI_GRAPH_LOOP) && !prof;
  if (graph_loop) {
    s = loop_graph(g, blocks, mode, async);
    if (s != DI_OK) return s;
  }
  while (!converged && launched < max_sweeps) {
    const int64_t k = graph_loop ? 0 : std::min<int64_t>(batch, max_sweeps - launched);
    const int64_t sweeps_before = g.sc_host->sweeps;
    const int64_t ev_per = 2 * blocks + 1;
    if (graph_loop) {  // the whole remaining loop on the device, one launch
      DI_CK(cudaGraphLaunch(g.loop_exec, g.stream));
    }
    for (int64_t j = 0; j < k; j++) {
      for (int b = 0; b < blocks; b++) {
        if (prof) DI_CK(cudaEventRecord(evs.get(ev_per * j + 2 * b), g.stream));
        if (async) {
          if (prof) DI_CK(cudaEventRecord(evs.get(ev_per * j + 2 * b + 1), g.stream));
          launch_cycle(g, &launches);
          continue;
        }
        launch_select(g, 0, &launches, b, blocks);
        if (prof) DI_CK(cudaEventRecord(evs.get(ev_per * j + 2 * b + 1), g.stream));
        if (mode != MODE_PULL) launch_push(g, &launches, b, blocks);
        if (mode != MODE_PUSH) launch_pull(g, &launches);
      }
      if (prof) DI_CK(cudaEventRecord(evs.get(ev_per * j + 2 * blocks), g.stream));
    }
    launched += k;
    s = sync_scalars(g);
    if (s != DI_OK) return s;
    DI_CK(cudaGetLastError());
    const int64_t real = g.sc_host->sweeps - sweeps_before;
    if (graph_loop) {
      launched = g.sc_host->sweeps;
      launches += (real + 1) * g.loop_launches;
    }
    if (prof) {
      for (int64_t j = 0; j < real && j < k; j++) {
        for (int b = 0; b < blocks; b++) {
          float a = 0.f, c = 0.f;
          cudaEventElapsedTime(&a, evs.get(ev_per * j + 2 * b), evs.get(ev_per * j + 2 * b + 1));
          cudaEventElapsedTime(&c, evs.get(ev_per * j + 2 * b + 1),
                               evs.get(ev_per * j + 2 * b + 2));
          select_ms += a;
          push_ms += c;
          push_launches++;
        }
      }
    }
    if (g.sc_host->stop) {
      launch_reduce_F(g, &launches);
      s = sync_scalars(g);
      if (s != DI_OK) return s;
      resid = g.sc_host->resid;
      if (err_of(resid, g.sc_host->e) <= tol) {
        converged = true;
        break;
      }
      // prediction q+s said converged but the exact sum disagrees by rounding: continue
      const int32_t zero = 0;
      DI_CK(cudaMemcpyAsync(&g.sc->stop, &zero, 4, cudaMemcpyHostToDevice, g.stream));
      g.sc_host->stop = 0;
    }
    // batch size: predicted sweeps left from the observed decay rate of r
    const double r_now = g.sc_host->r;
    int64_t next = 8;
    if (real > 0 && r_now > 0.0 && r_prev > r_now) {
      const double rate = std::pow(r_now / r_prev, 1.0 / (double)real);
      const double target = paper ? tol * (1.0 - d) : tol;
      if (rate < 1.0 && rate > 0.0) {
        const double left = std::log(target / r_now) / std::log(rate);
        next = (int64_t)std::ceil(std::max(1.0, left));
      }
    }
    batch = std::max<int64_t>(1, std::min<int64_t>(next, blocks > 1 ? 8 : 32));
    r_prev = r_now;
  }
  if (!converged || launched == 0) {
    launch_reduce_F(g, &launches);
    s = sync_scalars(g);
    if (s != DI_OK) return s;
    resid = g.sc_host->resid;
    converged = err_of(resid, g.sc_host->e) <= tol;
  }
  DI_CK(cudaEventRecord(t1, g.stream));
  DI_CK(cudaEventSynchronize(t1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  DI_CK(cudaGetLastError());
  g.solved = true;
  g.last_d = d;
  if (async) report_cycle_times(g, g.sc_host->sweeps);
  g.log_n = std::min<int64_t>(g.sc_host->sweeps, kLogCap);
  if (st) {
    const Scalars &c = *g.sc_host;
    memset(st, 0, sizeof(*st));
    st->sweeps = c.sweeps;
    st->selected_total = c.selected_total;
    st->link_diffusions = c.links_total;
    st->starvation_fallbacks = c.guards;
    st->nodes_scanned = c.scanned_total;
    st->pull_sweeps = c.pull_sweeps;
    st->gpu_launches = launches;
    st->residual_l1 = resid;
    st->dangling_absorbed = c.e;
    st->equivalent_iterations = g.l_global > 0 ? (double)c.links_total / (double)g.l_global : 0.0;
    st->solve_ms = ms;
    // algorithmic bytes
    st->counted_bytes = 12.0 * c.scanned_total + 40.0 * c.selected_total + 20.0 * c.links_total;
    st->push_bytes = 16.0 * c.selected_nd_total + 20.0 * c.links_total;
    st->push_ms = push_ms;
    st->select_ms = select_ms;
    st->push_launches = push_launches;
    st->error_estimate = resid / (1.0 - d - d * c.e);
    st->converged = converged ? 1 : 0;
    st->variant = (int32_t)v;
  }
  return converged ? DI_OK : DI_NOT_CONVERGED;
}

di_status di_residual(di_graph h, double *l1_out, double *F_out) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "di_residual: NULL handle");
  if (g->partitioned) {  // collective: the global sum
    double l1 = 0.0;
    di_status s = dist_residual(*g, &l1);
    if (s != DI_OK) return s;
    if (l1_out) *l1_out = l1;
  } else {
    int64_t launches = 0;
    launch_reduce_F(*g, &launches);
    di_status s = sync_scalars(*g);
    if (s != DI_OK) return s;
    if (l1_out) *l1_out = g->sc_host->resid;
  }
  if (F_out) {
    if (g->reordered)
      gather(*g, F_out, g->F - g->lo, g->new_of + g->lo);
    else
      DI_CK(cudaMemcpyAsync(F_out, g->F, (size_t)g->n * 8, cudaMemcpyDeviceToDevice, g->stream));
    DI_CK(cudaStreamSynchronize(g->stream));
  }
  return DI_OK;
}

di_status di_history(di_graph h, double *H_out) {
  Graph *g = (Graph *)h;
  if (!g || !H_out) return fail(DI_EINVAL, "di_history: NULL argument");
  if (g->reordered)
    gather(*g, H_out, g->H - g->lo, g->new_of + g->lo);
  else
    DI_CK(cudaMemcpyAsync(H_out, g->H, (size_t)g->n * 8, cudaMemcpyDeviceToDevice, g->stream));
  DI_CK(cudaStreamSynchronize(g->stream));
  return DI_OK;
}

di_status di_sweep_log(di_graph h, double *r, int64_t *selected, int64_t *links, uint8_t *mode,
                       int64_t cap, int64_t *n_out) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "di_sweep_log: NULL handle");
  const int64_t n = std::min<int64_t>(g->log_n, std::max<int64_t>(cap, 0));
  if (n > 0) {
    if (r) DI_CK(cudaMemcpy(r, g->log_r, (size_t)n * 8, cudaMemcpyDeviceToHost));
    if (selected) DI_CK(cudaMemcpy(selected, g->log_sel, (size_t)n * 8, cudaMemcpyDeviceToHost));
    if (links) DI_CK(cudaMemcpy(links, g->log_links, (size_t)n * 8, cudaMemcpyDeviceToHost));
    if (mode) DI_CK(cudaMemcpy(mode, g->log_mode, (size_t)n, cudaMemcpyDeviceToHost));
  }
  if (n_out) *n_out = n;
  return DI_OK;
}

// ------------------------------------------------------------------ test exports
di_status di_test_bins(int32_t out[4]) {
  if (!out) return fail(DI_EINVAL, "NULL");
  out[0] = kBinT;
  out[1] = kBinG;
  out[2] = kBinW;
  out[3] = kChunk;
  return DI_OK;
}

di_status di_test_perm(di_graph h, int32_t *old_of) {
  Graph *g = (Graph *)h;
  if (!g || !old_of) return fail(DI_EINVAL, "NULL argument");
  if (!g->reordered) {
    for (int64_t k = 0; k < g->n; k++) old_of[k] = (int32_t)k;
    return DI_OK;
  }
  DI_CK(cudaMemcpy(old_of, g->old_of, (size_t)g->n * 4, cudaMemcpyDeviceToHost));
  return DI_OK;
}

di_status di_test_csr(di_graph h, int64_t *row_ptr, int32_t *col, int32_t *deg, int32_t *kloop,
                      int64_t *csc_ptr, int32_t *csc_row) {
  Graph *g = (Graph *)h;
  if (!g) return fail(DI_EINVAL, "NULL handle");
  const size_t n = (size_t)g->n, l = (size_t)g->l;
  if (row_ptr) DI_CK(cudaMemcpy(row_ptr, g->row_ptr, (n + 1) * 8, cudaMemcpyDeviceToHost));
  if (col && l) DI_CK(cudaMemcpy(col, g->col, l * 4, cudaMemcpyDeviceToHost));
  if (deg) DI_CK(cudaMemcpy(deg, g->deg, n * 4, cudaMemcpyDeviceToHost));
  if (kloop) DI_CK(cudaMemcpy(kloop, g->kloop, n * 4, cudaMemcpyDeviceToHost));
  if (csc_ptr || csc_row) {
    if (!g->has_csc) return fail(DI_ESTATE, "di_test_csr: CSC not built (DI_BUILD_CSC)");
    if (csc_ptr) DI_CK(cudaMemcpy(csc_ptr, g->csc_ptr, (n + 1) * 8, cudaMemcpyDeviceToHost));
    if (csc_row && l) DI_CK(cudaMemcpy(csc_row, g->csc_row, l * 4, cudaMemcpyDeviceToHost));
  }
  return DI_OK;
}

di_status di_test_cycle(di_graph h, const double *F_in, const double *H_in, double r, double d,
                        di_variant v, double *T_out, double *v_out, double scal[3], int64_t counts[2],
                        double *F_out, double *H_out) {
  Graph *gp = (Graph *)h;
  if (!gp || !F_in || !H_in) return fail(DI_EINVAL, "di_test_cycle: NULL argument");
  if (v != DI_SOP && v != DI_CYC) return fail(DI_EINVAL, "di_test_cycle: DI_SOP or DI_CYC");
  Graph &g = *gp;
  if (g.partitioned) return fail(DI_EINVAL, "di_test_cycle: single-GPU graphs only");
  AllocScope as(g.stream);
  {
    di_status ps = prepare_cycle(g, false);
    if (ps != DI_OK) return ps;
  }
  const size_t n = (size_t)g.n;
  std::vector<int32_t> old_of;
  std::vector<double> Fi(n), Hi(n);
  if (g.reordered) {
    old_of.resize(n);
    DI_CK(cudaMemcpy(old_of.data(), g.old_of, n * 4, cudaMemcpyDeviceToHost));
  }
  for (size_t k = 0; k < n; k++) {
    const size_t u = g.reordered ? (size_t)old_of[k] : k;
    Fi[k] = F_in[u];
    Hi[k] = H_in[u];
  }
  DI_CK(cudaMemcpy(g.F, Fi.data(), n * 8, cudaMemcpyHostToDevice));
  DI_CK(cudaMemcpy(g.H, Hi.data(), n * 8, cudaMemcpyHostToDevice));
  double *rec = nullptr;
  DI_CK(dmalloc(&rec, 2 * n * 8 + 16));
  DI_CK(cudaMemsetAsync(rec, 0, 2 * n * 8 + 16, g.stream));
  {
    Scalars &s = *g.sc_host;
    const uint32_t epoch = s.epoch ? s.epoch : 1;
    memset(&s, 0, sizeof(Scalars));
    s.epoch = epoch;
    s.r = r;
    s.d = d;
    s.alpha = g.alpha;
    s.tol = 1e-300;
    s.variant = (int32_t)v;
  }
  DI_CK(cudaMemcpyAsync(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice, g.stream));
  int64_t launches = 0;
  launch_cycle_test(g, rec, rec + n, &launches);
  di_status s = sync_scalars(g);
  if (s != DI_OK) {
    dfree(rec);
    return s;
  }
  DI_CK(cudaGetLastError());
  std::vector<double> Tr(n), vr(n), Fo(n), Ho(n);
  DI_CK(cudaMemcpy(Tr.data(), rec, n * 8, cudaMemcpyDeviceToHost));
  DI_CK(cudaMemcpy(vr.data(), rec + n, n * 8, cudaMemcpyDeviceToHost));
  DI_CK(cudaMemcpy(Fo.data(), g.F, n * 8, cudaMemcpyDeviceToHost));
  DI_CK(cudaMemcpy(Ho.data(), g.H, n * 8, cudaMemcpyDeviceToHost));
  dfree(rec);
  for (size_t k = 0; k < n; k++) {
    const size_t u = g.reordered ? (size_t)old_of[k] : k;
    if (T_out) T_out[u] = Tr[k];
    if (v_out) v_out[u] = vr[k];
    if (F_out) F_out[u] = Fo[k];
    if (H_out) H_out[u] = Ho[k];
  }
  const Scalars &c = *g.sc_host;
  if (scal) {
    scal[0] = c.q;
    scal[1] = c.s;
    scal[2] = c.e_sw;
  }
  if (counts) {
    counts[0] = c.selected_total;
    counts[1] = c.links_total;
  }
  return DI_OK;
}

di_status di_test_select(di_graph h, const double *F_in, const double *H_in, double r, double d,
                         di_variant v, int32_t *ids, double *vals, int32_t *chunk, int64_t cap,
                         int64_t bin_off[5], double scal[3], int64_t counts[2], double *F_out,
                         double *H_out) {
  Graph *gp = (Graph *)h;
  if (!gp || !F_in || !H_in) return fail(DI_EINVAL, "di_test_select: NULL argument");
  if (v != DI_SOP && v != DI_CYC) return fail(DI_EINVAL, "di_test_select: DI_SOP or DI_CYC");
  Graph &g = *gp;
  const size_t n = (size_t)g.n;
  std::vector<int32_t> old_of;
  if (g.reordered) {
    old_of.resize(n);
    DI_CK(cudaMemcpy(old_of.data(), g.old_of, n * 4, cudaMemcpyDeviceToHost));
    std::vector<double> Fi(n), Hi(n);
    for (size_t k = 0; k < n; k++) {
      Fi[k] = F_in[old_of[k]];
      Hi[k] = H_in[old_of[k]];
    }
    DI_CK(cudaMemcpy(g.F, Fi.data(), n * 8, cudaMemcpyHostToDevice));
    DI_CK(cudaMemcpy(g.H, Hi.data(), n * 8, cudaMemcpyHostToDevice));
  } else {
    DI_CK(cudaMemcpy(g.F, F_in, n * 8, cudaMemcpyHostToDevice));
    DI_CK(cudaMemcpy(g.H, H_in, n * 8, cudaMemcpyHostToDevice));
  }
  {
    Scalars &s = *g.sc_host;
    const uint32_t epoch = s.epoch ? s.epoch : 1;
    memset(&s, 0, sizeof(Scalars));
    s.epoch = epoch;
    s.r = r;
    s.d = d;
    s.alpha = g.alpha;
    s.tol = 1e300;
    s.variant = (int32_t)v;
  }
  DI_CK(cudaMemcpy(g.sc, g.sc_host, sizeof(Scalars), cudaMemcpyHostToDevice));
  int64_t launches = 0;
  launch_select(g, 1, &launches);
  launch_finalize(g, &launches);
  di_status s = sync_scalars(g);
  if (s != DI_OK) return s;
  DI_CK(cudaGetLastError());
  const Scalars &c = *g.sc_host;
  int64_t off = 0;
  for (int b = 0; b < kBins; b++) {
    if (bin_off) bin_off[b] = off;
    off += c.bin_count[b];
  }
  if (bin_off) bin_off[kBins] = off;
  if (off > cap) return fail(DI_EINVAL, "di_test_select: cap too small");
  // bin contents, sorted by (node id, chunk) inside each bin (the tile order inside a bin is
  // the reservation order and carries no meaning)
  std::vector<int64_t> rp((size_t)g.n + 1);
  DI_CK(cudaMemcpy(rp.data(), g.row_ptr, ((size_t)g.n + 1) * 8, cudaMemcpyDeviceToHost));
  off = 0;
  for (int b = 0; b < kBins; b++) {
    const size_t m = (size_t)c.bin_count[b];
    std::vector<Entry> ent(m);
    std::vector<int32_t> eid(m);
    if (m) {
      DI_CK(cudaMemcpy(ent.data(), g.fr.ent[b], m * sizeof(Entry), cudaMemcpyDeviceToHost));
      DI_CK(cudaMemcpy(eid.data(), g.fr.id[b], m * 4, cudaMemcpyDeviceToHost));
    }
    std::vector<int32_t> uid(m);   // caller's numbering
    for (size_t k = 0; k < m; k++) uid[k] = g.reordered ? old_of[eid[k]] : eid[k];
    std::vector<size_t> order(m);
    for (size_t k = 0; k < m; k++) order[k] = k;
    std::sort(order.begin(), order.end(), [&](size_t x, size_t y) {
      if (uid[x] != uid[y]) return uid[x] < uid[y];
      return (ent[x].bl & kBegMask) < (ent[y].bl & kBegMask);
    });
    for (size_t k = 0; k < m; k++) {
      const size_t slot = order[k];
      const int32_t id = eid[slot];
      const int64_t beg = (int64_t)(ent[slot].bl & kBegMask);
      if (ids) ids[off] = uid[slot];
      if (vals) vals[off] = ent[slot].v;
      if (chunk) chunk[off] = (int32_t)((beg - rp[id]) / kChunk);
      off++;
    }
  }
  if (scal) {
    scal[0] = c.q;
    scal[1] = c.s;
    scal[2] = c.e_sw;
  }
  if (counts) {
    counts[0] = c.selected_total;
    counts[1] = c.links_total;
  }
  std::vector<double> Fo(n), Ho(n);
  DI_CK(cudaMemcpy(Fo.data(), g.F, n * 8, cudaMemcpyDeviceToHost));
  DI_CK(cudaMemcpy(Ho.data(), g.H, n * 8, cudaMemcpyDeviceToHost));
  for (size_t k = 0; k < n; k++) {
    const size_t u = g.reordered ? (size_t)old_of[k] : k;
    if (F_out) F_out[u] = Fo[k];
    if (H_out) H_out[u] = Ho[k];
  }
  return DI_OK;
}

}  // extern "C"
