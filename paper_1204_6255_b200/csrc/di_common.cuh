// di_common.cuh — internal types shared by the libdi.so translation units.
// Product code: nothing here is shared with oracle/ (which is independent C).
#pragma once
#include <vector>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/di.h"

namespace di {

// ----------------------------------------------------------------- tuning constants
// Select / compact (SURVEY §8(a) a3+a4): one tile = kSelThreads x kSelItems consecutive nodes.
constexpr int kSelThreads = 256;
constexpr int kSelItems = 4;
constexpr int kSelTile = kSelThreads * kSelItems;
// Degree bins of the push (north_star item 3):
//   T: 1..kBinT links -> one thread per node
//   G: kBinT+1..kBinG -> 8-lane group per node
//   W: kBinG+1..kBinW -> one warp per node
//   C: > kBinW        -> rows split in chunks of kChunk links, one warp per chunk
constexpr int kBins = 4;
constexpr int kBinT = 8;
constexpr int kBinG = 32;
constexpr int kBinW = 1024;
constexpr int kChunk = 1024;
constexpr int kPushThreads = 256;
constexpr int kRedThreads = 512;
constexpr int kLogCap = 1 << 16;  // per-sweep trace capacity
constexpr int kMaxSlices = 4096;   // finaliser slices (= push/pull grid size, <= this)
constexpr int kMaxBlocks = 256;    // block-ordered sweeps: sub-sweeps per cycle
// Skewed in-degrees (async.cu): when the top node takes more than kReplShare of the links, the
// kHotRanks hottest nodes are placed first and their REDs spread over replicated accumulators.
#ifndef DI_HOT_RANKS
#define DI_HOT_RANKS 64
#endif
constexpr int kHotRanks = DI_HOT_RANKS;
#ifndef DI_HOT_COPIES
#define DI_HOT_COPIES 16
#endif
constexpr int kRepCopies = DI_HOT_COPIES;  // copies of each hot accumulator (chosen by warp)
constexpr int kRepStride = 16;             // doubles between accumulators: one 128-B line each
constexpr double kReplShare = 0.0005;
// Warm tier (async.cu): on a skewed graph the kWarmIds ranks after the hot ones are
// placed one every 2^shift ids, and every CTA of k_cycle accumulates its pushes to them (and to the
// hot ids) in shared memory, flushed into F once when the CTA leaves the cycle.
constexpr int kWarmIds = -1;   // option "warm" default: auto (as many as fit in shared memory)
constexpr double kWarmShare = 0.10;   // auto: on when the hot + warm ranks take this share of the
constexpr double kWarmLinks = 32.0;    // links and L >= kWarmLinks x grid x slots

// Cold bins (async.cu): on one GPU, when F is larger than kColdF_L2 times the L2,
// the relabelling puts a first tier of kColdHotL2 x L2 bytes of nodes (by in-degree) right after
// the hot ids; REDs to them stay in L2, and a push to a node beyond them (a "cold" target: mostly
// an L2 miss, ~22 G random REDs/s into 1 GB) is appended as a 16-B record to the bin of its
// slice of 2^shift nodes (at most kColdBins slices), then applied slice by slice after the cycle
// (k_cold_apply: the slice's F lines stay in L2 while its records stream through).
constexpr int kPipeChunks = 8;                // pipelined host upload: source-id chunks (graph_build.cu)
constexpr int64_t kPipeMinLinks = 1ll << 22;  // ... for link lists of at least this many links
constexpr int kColdBins = 64;
constexpr int kColdChunk = 64;          // records per warp chunk (one 1 KB run of a bin)
constexpr double kColdF_L2 = 2.0;
constexpr double kColdHotL2 = 0.5;
constexpr int kColdMinShift = 16;
struct __align__(16) ColdRec {
  int32_t j;     // internal target id (-1: none)
  int32_t pad;
  double v;
};

enum BinId { BIN_T = 0, BIN_G = 1, BIN_W = 2, BIN_C = 3 };

// Pull (CSC) variant, SURVEY §8(a) a5': static bins of target rows by in-degree.
//   P0: 1..kPullT in-links -> one thread per row
//   P1: ..kPullG           -> 8-lane group per row
//   P2: ..kPullChunk       -> one warp per row
//   P3: > kPullChunk       -> rows split in kPullChunk chunks, one warp each (partial sums
//                             added with an fp64 atomic; every other row is a plain RMW)
constexpr int kPullBins = 4;
constexpr int kPullT = 8;
constexpr int kPullG = 128;
constexpr int kPullChunk = 8192;
struct __align__(16) PullEntry {
  int64_t beg;   // first in-link (csc_row index)
  int32_t len;   // in-links in this entry
  int32_t j;     // target node (local id)
};
enum SweepMode { MODE_PUSH = 0, MODE_PULL = 1, MODE_AUTO = 2 };

// Multi-GPU: rank g owns the node range [b[g], b[g+1]) (caller's numbering, and
// internal numbering after the per-range relabelling).
constexpr int kMaxWorld = 16;
// Peer-memory inbox of a partitioned graph (dist.cu): per sender a segment of kRingSlots * icap
// 12-byte records (synchronous sweeps use slots 0/1 by sweep parity; DI_DIST_ASYNC uses the
// segment as a ring), then one 256-B control line per sender (its published ring tail).
constexpr int kRingSlots = 4;
struct DistBounds {
  int world;
  int64_t b[kMaxWorld + 1];
};

// Process-wide tuning / diagnostic options (di_set_option, include/di.h). Upload-time options are
// copied into each graph by di_graph_upload; the rest are read when used.
struct Options {
  int red_hint = 1;          // "red_hint": L2 evict_last policy on the push's REDs into F
  int push_occ = 4;          // "push_occ": k_push resident blocks per SM
  double auto_ratio = 0.35;  // "auto_ratio": DI_AUTO pulls a sweep with links(S) > ratio * L
  int stripes = 0;           // "stripes": relabelling stripes (0 auto, 1 plain degree order)
  int hot_acc = 1;           // "hot_acc": replicated accumulators for the hottest targets
  double repl_share = kReplShare;  // "repl_share": top in-degree share that turns them on
  int cold_bins = -1;        // "cold_bins": -1 auto (F > 2 L2), 0 off, 1 on (one GPU, DI_ASYNC)
  int64_t cold_tier = 0;     // "cold_tier": first-tier size in nodes (0: half the L2 in bytes)
  int cycle_grid_div = 1;    // "cycle_grid_div": 1/k of k_cycle's grid (emulated-rank studies)
  int cycle_times = 0;       // "cycle_times": per-CTA start/end times of each cycle (stderr)
  int p2p = 1;               // "p2p": peer-memory inboxes for the partitioned exchange
  int p2p_force = 0;         // "p2p_force": create the inbox on a one-rank communicator too
  int build_trace = 0;       // "build_trace": host timestamps of the build phases (stderr)
  int remote_compact = 1;    // "remote_compact": hot remote accumulator + cold records (P2P)
  int64_t remote_tier = 0;   // "remote_tier": hot remote targets per range (0: auto)
  int long_lanes = 1;        // "long_lanes": k_cycle long rows with lane-consecutive targets
  int row_sort = 0;          // "row_sort": one-GPU build by counting sort + segmented row sort
  int line_spread = 16;      // "line_spread": nodes of one rank class per 16-node line (1, 2, 4, 8, 16)
  int cold_shift = 0;        // "cold_shift": cold-bin slices of 2^shift nodes (0: auto, <= kColdBins bins)
  int warm = kWarmIds;       // "warm": ranks after the hot ones accumulated in shared memory by k_cycle
                             // (skewed graphs; -1 auto, 0 off)
  int warm_flush = 0;        // "warm_flush": k_cycle flushes them every k tiles of a CTA (0: at its end)
  int warm_shift = 0;        // "warm_shift": warm ranks every 2^k ids (0: spread over the range / first tier)
  int dist_parts = 1;        // "dist_parts": partitioned DI_ASYNC: each cycle in k parts, an exchange after each
};
Options options();           // a snapshot of the current options

// Device-resident sweep state. Every field is written only by the "last block" of the
// select kernel (the finaliser) or by the host between solves, so kernels never race on it.
struct __align__(256) Scalars {
  double r;          // r_n: threshold fluid for the current sweep (sum F at sweep start)
  double e;          // cumulative dangling absorption
  double q, s, e_sw; // last sweep: unselected fluid, pushed fluid, dangling absorbed
  double resid;      // exact sum F from the reduce kernel
  double d, tol;     // solve parameters (device-resident: kernels take constant arguments)
  int32_t variant, paper_err, trace, mode;  // mode: SweepMode
  int64_t pull_thr;  // DI_AUTO: a sweep with more than pull_thr links runs in pull mode
  unsigned long long fill_links[32];  // DI_AUTO: links of the current frontier (own line)
  int32_t stop;      // 1: convergence reached after the current sweep's push
  int32_t guard;     // 1: next sweep runs with threshold 0 (starvation guard, reading G5)
  int32_t active;    // 1: the current sweep emitted push work
  int32_t pull;      // 1: the current sweep runs in pull mode (dense S vector)
  uint32_t epoch;    // select-launch counter: tags look-back flags, starts at 1
  uint32_t ticket;   // last-block detection of the select kernel
  uint32_t red_ticket;
  uint32_t pad0;
  int64_t bin_count[kBins];  // entries in each bin for the current sweep (read by the push)
  unsigned long long bin_fill[kBins][32];  // reservation counters (one 256-B line each)
  int64_t sweep_sel, sweep_links, sweep_sel_nd;
  int64_t sweeps, selected_total, selected_nd_total, links_total, scanned_total, guards,
      pull_sweeps;
  double r_run;              // block-ordered sweeps: running sum F inside a cycle
  int64_t sel_cyc, links_cyc;
  int64_t max_sweeps;        // DI_GRAPH_LOOP: the device-side loop stops at this many sweeps
  unsigned int tile_next;    // DI_ASYNC: next tile of the cycle (dynamic, increasing order)
  unsigned int hub_flag;     // DI_ASYNC hub items: tile 0 published hv[] for cycle hub_want + 1
  unsigned int hub_want;     //   (advanced by the last CTA of every cycle)
  double alpha;              // DI-SOP threshold scale (di_set_threshold_scale; 1 = P:298)
  // partitioned sweeps, counted on the device by k_dist_finalize (the batched peer-memory loop
  // reads them once per batch): entries this rank sent, all ranks' entries of the last sweep,
  // sweeps whose lists went through peer memory
  int64_t x_entries, x_lists_last, x_p2p, x_cold;
};

// One push work item: a row (or a kChunk-link chunk of a hub row) of a selected node.
// bl = first link index (48 bits) | number of links (16 bits); v = T_i*d/#out_i ("sent").
struct __align__(16) Entry {
  uint64_t bl;
  double v;
};
constexpr int kLenShift = 48;
constexpr uint64_t kBegMask = (1ull << kLenShift) - 1;

// Frontier: one contiguous array per degree bin. Each select tile reserves a contiguous range
// of a bin with one atomicAdd and writes its entries there in ascending node order; the order
// of tiles inside a bin is the (nondeterministic) reservation order, which the push does not
// depend on (its fp64 atomics are order-nondeterministic anyway).
struct Frontier {
  Entry *ent[kBins];
  int32_t *id[kBins];            // node id of each entry (self-loop test, tests)
  int64_t cap[kBins];            // static capacity: rows (chunks for C) with a degree in the bin
};

struct Graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t n = 0;          // nodes owned (== global n on one GPU)
  int64_t n_global = 0;
  int64_t lo = 0, hi = 0; // owned global range
  int64_t l = 0;          // links kept (local)
  int64_t l_global = 0;
  bool has_loops = false;
  bool has_csc = false;
  int push_occ = 4;         // k_push min blocks per SM (option push_occ)
  int red_hint = 1;         // L2 evict_last hint on the push's REDs into F (option red_hint)
  int rank = 0, world = 1;
  bool partitioned = false;  // built with a communicator (dist.cu path), even of one rank
  bool local_links = false;  // DI_LOCAL_LINKS: this rank's links only, range [local_lo, local_hi)
  int64_t local_lo = 0, local_hi = 0;
  std::vector<char *> inbox;  // fused exchange: every rank's inbox as mapped here (dist.cu)
  int64_t icap = 0;          // records per inbox segment (largest owned range)
  bool p2p = false;          // the inbox exists: k_compact_remote writes through peer memory
  double e_global = 0.0, e_cycle = 0.0;  // DI_DIST_ASYNC: global absorption (resume; last meeting)
  unsigned long long *ring = nullptr;  // DI_DIST_ASYNC state: tsent, head, snap [kMaxWorld each],
                                       // then 8 doubles (sent, applied, r_loc, r_loc_sync, r_sync)
  // locality relabelling: internal id = new_of[user id]; user id = old_of[internal id]
  bool reordered = false;
  int stripes = 0;           // relabelling stripes (option stripes; 0 = auto: stripes of ~1024 nodes,
                             // 1 = plain degree order)
  int64_t hot_count = 0;     // skewed graphs: the hot_count hottest nodes are internal ids 0..
  double alpha = 1.0;        // DI-SOP threshold scale
  double repl_share = kReplShare;  // top in-degree share that turns hot placement on (option repl_share)
  int hot_acc = 1;           // replicated accumulators for the hottest targets, every single-GPU
                             // push schedule and PI' (option hot_acc)
  int grid_div = 1;          // option cycle_grid_div
  int cycle_times = 0;       // option cycle_times
  int p2p_opt = 1, p2p_force = 0;  // options p2p, p2p_force
  double *rep = nullptr;     // replicated accumulators, then hv[kHotRanks] (async.cu)
  unsigned long long *cyc_times = nullptr;  // option cycle_times: per-CTA start/end per cycle
  int64_t *hub_items = nullptr;  // DI_ASYNC hub items: (row, first link, end link) triples
  int n_hub = 0;
  int64_t max_indeg = 0;     // largest in-degree (set by the relabelling pass)
  // cold bins (async.cu): internal ids >= cold_lo are cold (cold_lo == n: off)
  int cold_mode = -1;        // -1 auto (F > kColdF_L2 x L2), 0 off, 1 on (di_set_option)
  int64_t cold_tier = 0;     // > 0: first-tier size in nodes instead of kColdHotL2 x L2 / 8
  int64_t l2_bytes = 0;
  int64_t cold_lo = INT64_MAX;
  int cold_shift = 0, cold_nbins = 0;
  ColdRec *cold_rec = nullptr;     // arena: bin b's region starts at record cold_off[b]
  int64_t *cold_off = nullptr;     // device [kColdBins + 1]
  unsigned long long *cold_top = nullptr;  // device: records reserved per bin (one line each)
  int32_t *cold_fill = nullptr;    // device: records written per chunk, chunk k of the arena
  int32_t *new_of = nullptr, *old_of = nullptr;
  double *Bperm = nullptr;   // B in internal order (custom B)
  double *xfer = nullptr;    // scratch for permuted copies
  // CSR (sources owned), global column ids
  int64_t *row_ptr = nullptr;
  int32_t *col = nullptr;
  int32_t *deg = nullptr;
  int32_t *kloop = nullptr;
  // CSC (in-links of owned targets)
  int64_t *csc_ptr = nullptr;
  int32_t *csc_row = nullptr;
  // pull variant: static row entries per in-degree bin
  PullEntry *pe[kPullBins] = {nullptr, nullptr, nullptr, nullptr};
  int64_t pe_count[kPullBins] = {0, 0, 0, 0};
  PullEntry *re[kPullBins] = {nullptr, nullptr, nullptr, nullptr};  // PI' static out-rows
  int64_t re_count[kPullBins] = {0, 0, 0, 0};
  double *cmp_partials = nullptr;
  double auto_ratio = 0.35; // DI_AUTO threshold on links(S_n)/L (option auto_ratio)
  // state
  double *F = nullptr, *H = nullptr;
  double *S = nullptr;       // pull mode: dense per-node sent value
  double *aux = nullptr;     // comparators: x_new
  Scalars *sc = nullptr;     // device
  Scalars *sc_host = nullptr;  // pinned mirror
  double *partials = nullptr;  // per-tile q, s, e, taken partials (4 per tile)
  double *ppartials = nullptr; // per-slice reductions of the tile partials (finaliser level 1)
  int64_t *ipartials = nullptr;  // per-tile selected, selected non-dangling, links
  int64_t ntiles = 0;
  double *red_partials = nullptr;
  Frontier fr{};
  // trace
  double *log_r = nullptr;
  int64_t *log_sel = nullptr, *log_links = nullptr;
  uint8_t *log_mode = nullptr;
  int64_t log_n = 0;
  bool solved = false;
  double last_d = 0.85;
  // DI_GRAPH_LOOP: the sweep loop as a CUDA graph with a device-side while node (one cycle per
  // iteration), instantiated once per (blocks, mode) and replayed
  cudaGraphExec_t loop_exec = nullptr;
  cudaGraph_t loop_graph = nullptr;
  int loop_key = -1;
  int64_t loop_launches = 0;   // kernels per loop iteration
  // multi-GPU (dist.cu): partition, communicator and the per-sweep exchange buffers
  DistBounds bounds{1, {0}};
  struct Comm *comm = nullptr;
  struct Group *group = nullptr;
  double *R = nullptr;            // remote fluid accumulator, fp64[n_global], all-zero between sweeps
  double *sval = nullptr;         // send records: 12-byte (id, value), owner p's segment at b[p]
  unsigned long long *tcnt = nullptr;  // records per owner (one 256-B line each) + a ticket
  // per-sweep header of this rank, 8 + world int64 words: dsum (q, s, e, taken as fp64), isum
  // (selected, non-dangling, links, scanned), sendcnt (entries for each peer); one allgather per
  // sweep gives every rank all headers (global sums in rank order, its receive counts)
  int64_t *hdr = nullptr;
  int64_t *ghdr = nullptr;        // device: world headers after the allgather
  int64_t *ghdr_h = nullptr;      // pinned copy of ghdr
  int64_t *sendcnt = nullptr;     // views into hdr
  double *dsum = nullptr;
  int64_t *isum = nullptr;
  int32_t *rid = nullptr;         // received 12-byte records, capacity (world-1) * n
  // compact remote path (dist.cu, async.cu)
  int remote_compact = 1;         // option remote_compact
  int64_t remote_tier = 0;        // option remote_tier (0: auto)
  int64_t rtier[kMaxWorld] = {0}; // hot remote targets at the start of every range
  double *racc = nullptr;         // their accumulator, sum of rtier
  int64_t ccap = 0;               // cold records per (sender, parity) inbox region
  int64_t cwin = 0;               // owner window of the cold-target column encoding (dist.cu)
  size_t cold_off0 = 0, fill_off0 = 0;
  unsigned long long *ctop = nullptr;
  int32_t *ccol = nullptr;        // the CSR columns encoded for the compact path (dist.cu)
  bool R_ready = false;           // R (global-size accumulator) allocated: bulk / ring / send-recv
  int cur_par = 0, cur_compact = 0;  // solve_dist -> launch_cycle: inbox parity, compact path
  int long_lanes = 1;             // option long_lanes
  int row_sort = 0;               // option row_sort
  int line_spread = 16;           // option line_spread
  int cold_shift_opt = 0;         // option cold_shift
  int warm_opt = kWarmIds;        // option warm
  int64_t warm_count = 0;         // warm tier: ranks hot_count.. placed at hot_count + k << warm_shift
  int warm_shift = 0;
  int warm_flush = 0;             // option warm_flush
  int warm_shift_opt = 0;         // option warm_shift
  int dist_parts = 1, cur_part = -1;  // option dist_parts; the part solve_dist launches next
                                      // (-1: whole cycles, every other caller)
};

// ---------------------------------------------------------------- device memory
// Every device buffer of the library comes from the device's default stream-ordered pool
// (cudaMallocAsync) on the calling handle's stream, with the pool's release threshold raised so
// that memory freed by one upload / solve is reused by the next without cudaMalloc/cudaFree
// (which synchronise the device and cost ms per GB). API entry points set the stream with
// AllocScope; dmemset is the stream-ordered memset on the same stream.
cudaStream_t &alloc_stream();
struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~AllocScope() { alloc_stream() = prev; }
};
cudaError_t dmalloc_bytes(void **p, size_t bytes);
template <typename T>
inline cudaError_t dmalloc(T **p, size_t bytes) {
  return dmalloc_bytes(reinterpret_cast<void **>(p), bytes);
}
void dfree(void *p);
cudaError_t pinned_scalars_get(Scalars **out);   // pinned host mirror of a graph's Scalars
void pinned_scalars_put(Scalars *p);
cudaError_t dmemset(void *p, int v, size_t bytes);

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string &msg);
#define DI_CK(call)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ::di::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));              \
      return e_ == cudaErrorMemoryAllocation ? DI_ENOMEM : DI_ECUDA;                    \
    }                                                                                   \
  } while (0)

// ---------------------------------------------------------------- launchers
// graph_build.cu
void btrace(const char *what);   // option build_trace: host timestamp of a build phase (stderr)
di_status build_graph(Graph &g, const int32_t *src, const int32_t *dst, int64_t n_links,
                      uint32_t flags);
// diffusion.cu
int64_t select_tiles(int64_t n);
di_status alloc_state(Graph &g);
void launch_init(Graph &g, const double *B, double d, int64_t *launches);
void launch_reduce_F(Graph &g, int64_t *launches);
void launch_reduce_F_setr(Graph &g, int64_t *launches);
void launch_select(Graph &g, int test_mode, int64_t *launches, int blk = 0, int blocks = 1);
void launch_push(Graph &g, int64_t *launches, int blk = 0, int blocks = 1);
void launch_finalize(Graph &g, int64_t *launches);
void launch_pull(Graph &g, int64_t *launches);
void launch_loop_cond(Graph &g, cudaGraphConditionalHandle h);
// async.cu
void report_cycle_times(Graph &g, int64_t cycles);
void launch_cycle(Graph &g, int64_t *launches);
void launch_cycle_test(Graph &g, double *rec_T, double *rec_v, int64_t *launches);
di_status prepare_cycle(Graph &g, bool async);
di_status alloc_pull(Graph &g);
di_status build_bin_entries(Graph &g, const int64_t *ptr, int64_t n, PullEntry **out, int64_t *counts);
di_status alloc_dist(Graph &g);
int64_t cycle_warps(const Graph &g);
int warm_fit();
// dist.cu
di_status solve_dist(Graph &g, double d, const double *B, double tol, int variant,
                     int64_t max_sweeps, uint32_t flags, di_stats *st);
di_status dist_residual(Graph &g, double *l1);
void free_dist(Graph &g);
// comparators.cu
di_status run_comparator(Graph &g, double d, double tol, int variant, int64_t max_sweeps,
                         uint32_t flags, di_stats *st);

}  // namespace di
