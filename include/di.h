/* include/di.h — C ABI of the B200-native D-iteration library (libdi.so).
 *
 * What it computes. The fixed point X = P.X + B of PAPER.md §1 for the
 * PageRank instantiation of §2.5: for every link i -> j of the link list,
 * P_ji = d / #out_i (#out_i counts every listed link of i, duplicates included),
 * dangling columns (#out_i = 0) are zero, and a node with k self-loop copies folds its
 * self-return series (generalised to k copies: DESIGN.md reading G6).
 * The solver is the D-iteration fluid diffusion (§2.5.4 DI-CYC P:249-284, §2.5.5 DI-SOP
 * P:286-299) reformulated as bulk-synchronous frontier sweeps (R1): it reaches
 * the same fixed point as the paper's sequential loop, not bit-identical iterates.
 *
 * Conventions.
 *  - Every call returns di_status; DI_OK = 0, positive = warning with a valid state,
 *    negative = error (the handle is unchanged unless stated). di_last_error() returns a
 *    thread-local message for the last failure.
 *  - Pointers are device pointers unless a flag or the argument says "host".
 *  - The library never frees caller memory; a di_graph owns every device buffer it
 *    allocates, released by di_graph_free.
 *  - One handle per stream; calls on one handle are not thread-safe. All work is enqueued
 *    on the handle's stream; di_solve/di_residual/di_history/di_stats_* block until their
 *    results are available on the host.
 *  - There is no CPU fallback: a missing or unusable CUDA device yields DI_ECUDA.
 */
#ifndef DI_H
#define DI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct di_graph_s *di_graph;  /* opaque */

typedef enum {
  DI_OK = 0,
  DI_NOT_CONVERGED = 1, /* max_sweeps reached; state (F, H) valid and resumable */
  DI_EINVAL = -1,       /* bad argument (range, id out of [0,n), d not in (0,1), tol <= 0 ...) */
  DI_ENOMEM = -2,       /* device allocation failed */
  DI_ECUDA = -3,        /* CUDA runtime error (message in di_last_error) */
  DI_ENCCL = -4,        /* NCCL error (multi-GPU) */
  DI_ESTATE = -5        /* call not valid in the handle's state (e.g. DI_RESUME before a solve) */
} di_status;

/* Solver variants (§2.3). */
typedef enum {
  DI_SOP = 0,      /* D-iteration, select F_i > r_n * #out_i / L           */
  DI_CYC = 1,      /* D-iteration, select F_i > 0                               */
  DI_PI_PULL = 2,  /* comparator: power iteration per row, pull over in-links      */
  DI_PI_PUSH = 3,  /* comparator: power iteration per column, push over out-links  */
  DI_GS_BLOCK = 4  /* comparator: Gauss-Seidel, ordered node blocks (R4)  */
} di_variant;

/* di_graph_upload flags */
#define DI_DEDUP            0x1u  /* drop duplicate links (default keeps multiplicities)  */
#define DI_DROP_SELF_LOOPS  0x2u  /* drop i -> i links (default folds them)            */
#define DI_BUILD_CSC        0x4u  /* also build the in-link (CSC) index: pull variant, PI, GS     */
#define DI_HOST_PTRS        0x8u  /* src/dst are host pointers (copied inside the call)           */
#define DI_LOCAL_LINKS      0x10u /* partitioned: this rank passes only the links whose source is
                                     in its node range dist->lo..hi (caller's numbering; the
                                     ranges of the ranks must tile [0, n) in rank order); the
                                     in-degrees are summed across ranks. Without it every rank
                                     passes the full list and the library balances the ranges */
#define DI_NO_REORDER       0x20u /* keep the caller's node numbering internally (default relabels
                                     by descending in-degree for L2 locality; results are always
                                     returned in the caller's numbering)                          */

/* di_solve flags */
#define DI_PUSH         0x0u   /* push-only sweeps (default)                                       */
#define DI_PULL         0x1u   /* pull (CSC) sweeps for every sweep (needs DI_BUILD_CSC)           */
#define DI_AUTO         0x2u   /* per-sweep push/pull choice by predicted bytes (needs CSC)        */
#define DI_RESUME       0x4u   /* continue from the current (F, H) instead of F = B, H = 0         */
#define DI_PAPER_ERROR  0x8u   /* stop on sum(F)/(1-d-d*e) <= tol instead of sum(F)    */
#define DI_TRACE        0x10u  /* record the per-sweep log read by di_sweep_log                    */
#define DI_PROFILE      0x20u  /* time every kernel with CUDA events (fills *_ms fields)           */
#define DI_GRAPH_LOOP   0x40u  /* run the sweep loop as one CUDA graph: a while node whose body is
                                  one cycle + a condition kernel (!stop && sweeps < max_sweeps);
                                  one host launch and one synchronisation per solve (ignored with
                                  DI_PROFILE; single GPU)                                        */
#define DI_ASYNC        0x100u /* asynchronous cycles: one persistent kernel per cycle takes tiles
                                  of nodes in increasing order, selects against the cycle's r with
                                  the live F (the fluid read is taken by a RED F_i -= f) and pushes at once:
                                  the paper's cyclic order up to the concurrency of the
                                  grid; push only; on a partitioned graph every rank runs its
                                  range's cycle and the remote fluid is exchanged once per cycle;
                                  iterates not bit-reproducible                                 */
/* Exchange of remote fluid on a partitioned graph: by default each sweep
 * chooses by predicted bytes between the sparse (id, value) lists (12 B per touched remote
 * target) and the dense fallback, a per-owner reduction of the remote accumulator (8 B per remote
 * node: (G-1)/G * 8N per rank), taking the dense one when the last sparse sweep's lists were
 * larger; these flags force one of them. Ignored on one GPU. */
#define DI_XCHG_SPARSE  0x200u
#define DI_XCHG_DENSE   0x400u
/* The sparse lists are written by the compaction kernel straight into the owner's inbox through
 * peer memory (fused pack + transfer: NVLink stores into an NCCL symmetric window, or device
 * pointers of one GPU for an in-process group) when the upload could create the inboxes; this
 * flag moves them with the backend's send/recv instead. */
#define DI_XCHG_NOP2P   0x800u
/* Asynchronous multi-GPU cycles (with DI_ASYNC on a partitioned graph): no
 * collective between two cycles — each rank runs its cycles back to back, the remote fluid goes
 * through peer-memory rings drained at the start of every cycle, and the ranks meet every 4
 * cycles (drain, exact global sum F, stop test). Needs the peer-memory inboxes. */
#define DI_DIST_ASYNC   0x1000u
/* Block-ordered cycles (F1): each cycle visits K ordered blocks of
 * internal node ids; block b is selected against the cycle's threshold r (computed once per
 * cycle) with the live F, i.e. including the fluid pushed by blocks 0..b-1 this
 * cycle: the paper's cyclic order at block granularity. K in [2, 255]; push sweeps only;
 * 0 or 1 = the plain bulk sweep. Single GPU. */
#define DI_BLOCKS(K)    ((((uint32_t)(K)) & 0xFFu) << 16)

typedef struct {
  int64_t sweeps;               /* sweeps (bulk) or cycles (DI_BLOCKS, DI_ASYNC) executed, incl.
                                   starvation fallbacks                                           */
  int64_t selected_total;       /* sum over sweeps of |S_n| (diffused nodes, dangling included)  */
  int64_t link_diffusions;      /* sum over sweeps of sum_{i in S_n} #out_i         */
  int64_t starvation_fallbacks; /* sweeps that selected nothing and forced one DI-CYC sweep (G5) */
  int64_t nodes_scanned;        /* sum over sweeps of nodes tested by the select kernel          */
  int64_t pull_sweeps;          /* sweeps executed in pull (CSC) mode                            */
  int64_t gpu_launches;         /* kernels launched by this call                                  */
  double residual_l1;           /* ||F||_1 at exit (exact deterministic sum)                     */
  double dangling_absorbed;     /* e = sum of transit at dangling nodes           */
  double equivalent_iterations; /* link_diffusions / L ("nb iter")            */
  double solve_ms;              /* CUDA-event time of the whole call on the handle's stream      */
  double counted_bytes;         /* algorithmic bytes: all kernels          */
  double push_bytes;            /* algorithmic bytes of the push (a5) / pull (a5') kernels       */
  double push_ms;               /* DI_PROFILE: summed event time of the push/pull kernels        */
  double select_ms;             /* DI_PROFILE: summed event time of the select kernels           */
  double error_estimate;        /* sum(F)/(1-d-d*e); comparators: their own error        */
  int64_t push_launches;        /* DI_PROFILE: push/pull launches that did work                  */
  int32_t converged;            /* 1 if the stop test passed                                     */
  int32_t variant;
  double exchange_bytes;        /* multi-GPU: bytes this rank sent (12 per (remote id, sweep); dense
                                   sweeps: 8 per remote node)                                     */
  int64_t exchange_entries;     /* multi-GPU: (remote id, value) entries this rank sent           */
  double exchange_ms;           /* multi-GPU, DI_PROFILE: event time of list exchange + apply     */
  int64_t dense_exchanges;      /* multi-GPU: sweeps whose exchange took the dense fallback       */
  int64_t p2p_exchanges;        /* multi-GPU: sweeps whose lists went through peer memory (fused) */
  int64_t meetings;             /* DI_DIST_ASYNC: collective meetings (drain + global sum F)       */
  int64_t exchange_cold;        /* multi-GPU compact path: 16-B records of pushes to cold remote
                                   targets this rank wrote into the owners' inboxes (slots
                                   reserved); exchange_bytes = 12 entries + 16 cold (+ dense)     */
} di_stats;

/* In-process rank group: `world` emulated ranks, one host thread each, sharing one GPU. The
 * collectives become host barriers plus device-to-device copies (no kernel waits for another
 * rank). Used to run and test the partitioned path on a single GPU. */
typedef struct di_group_s *di_group;

/* Multi-GPU descriptor: one process per GPU with NCCL over NVLink/NVSwitch, or
 * one host thread per rank with a di_group. Every rank passes the FULL link list; rank g then
 * owns the node range [lo_g, hi_g) returned by di_graph_range (1-D, contiguous in the caller's
 * numbering, balanced on 20 B per link + 12 B per node), and each sweep exchanges the fluid sent
 * to remote targets as (id, value) lists (12 B per distinct remote target per sweep). */
typedef struct {
  int32_t rank, world;        /* 0 <= rank < world <= 16                                        */
  const void *nccl_unique_id; /* 128-byte ncclUniqueId, identical on every rank (host pointer),
                                 from di_nccl_unique_id on one rank; NULL with a group. Graphs
                                 uploaded with the same id share one NCCL communicator, kept
                                 until the process exits (an id initialises one communicator) */
  di_group group;             /* in-process group from di_group_create, else NULL                */
  int64_t lo, hi;             /* DI_LOCAL_LINKS: this rank's node range [lo, hi); else ignored   */
} di_dist;

/* Fill out128 (host, 128 bytes) with a fresh ncclUniqueId (call on one rank, broadcast the bytes,
 * e.g. with torch.distributed). NCCL is loaded at run time (libnccl.so.2, the copy torch loaded).
 * Errors: DI_ENCCL if NCCL cannot be loaded. */
di_status di_nccl_unique_id(void *out128);
/* Create / free an in-process group of `world` ranks (1..16). di_group_free fails with
 * DI_ESTATE while graphs built on the group are alive. */
di_status di_group_create(int32_t world, di_group *out);
di_status di_group_free(di_group grp);
/* Mark the group failed: every rank blocked in (or later entering) a group collective returns
 * DI_ESTATE instead of waiting for a rank that will not arrive. Call when one rank's call
 * failed; the group's graphs can then only be freed. */
di_status di_group_abort(di_group grp);

/* Build the device graph (§2.1, "Init" timed separately).
 *  src, dst : n_links int32 node ids of the links src[k] -> dst[k]; device pointers, or host
 *             pointers with DI_HOST_PTRS. Any order; caller keeps ownership.
 *  n_links  : >= 0.   n_nodes : in [1, 2^31 - 1].
 *  stream   : cudaStream_t the handle will use (NULL = legacy default stream).
 *  dist     : NULL for one GPU; otherwise every rank calls collectively with the same link list
 *             and owns the node range returned by di_graph_range (1-D partition).
 *             Partitioned graphs: no DI_BUILD_CSC (DI_EINVAL), n_nodes >= world; with DI_LOCAL_LINKS a
 *             link whose source lies outside dist->lo..hi, or ranges that do not tile [0, n), fail
 *             on every rank with DI_EINVAL.
 * Layout built in HBM: CSR row_ptr int64[n+1], col int32[L] sorted by (src, dst); deg int32[n];
 * kloop int32[n] (self-loop multiplicity); optional CSC (col_ptr int64[n+1], row int32[L]).
 * Errors: DI_EINVAL (sizes, an id outside [0, n): the message names the first bad index),
 * DI_ENOMEM, DI_ECUDA, DI_ENCCL. On error *out is NULL. */
di_status di_graph_upload(const int32_t *src, const int32_t *dst, int64_t n_links, int64_t n_nodes,
                          uint32_t flags, void *stream, const di_dist *dist, di_graph *out);

/* Process-wide tuning and diagnostic options. Every knob of the library is one of these (there are
 * no environment variables). Upload-time options (marked U) apply to graphs uploaded afterwards;
 * the others are read when used. Not for the inner loop: the call takes a mutex.
 *   name             default  range     meaning
 *   "red_hint"       1        0..1      U: L2 evict_last policy on the push's REDs into F
 *   "push_occ"       4        1..32     U: resident blocks per SM of the bulk push kernel
 *   "auto_ratio"     0.35     >= 0      U: DI_AUTO pulls a sweep whose links(S) exceed ratio * L
 *   "stripes"        0        >= 0      U: relabelling stripes (0: ~1024-node stripes, prime count;
 *                                          1: plain descending in-degree order)
 *   "hot_acc"        1        0..1      U: replicated accumulators for the 64 hottest targets
 *   "repl_share"     0.0005   0..1      U: top in-degree share of L that turns them on
 *   "cold_bins"      -1       -1..1     U: cold bins of DI_ASYNC on one GPU (-1: when F > 2 x L2;
 *                                          0 off; 1 on): pushes to targets beyond the first tier
 *                                          are binned by target slice and applied slice by slice
 *   "cold_tier"      0        >= 0      U: first-tier size in nodes (0: half the L2 in bytes)
 *   "cold_shift"     0        0..30     U: cold-bin slices of 2^shift nodes (0: about the L2 in F)
 *   "cycle_grid_div" 1        1..4096   U: DI_ASYNC grid divided by k (emulated-rank studies)
 *   "cycle_times"    0        0..1      U: per-CTA start/end times of each cycle, summary on stderr
 *   "p2p"            1        0..1      U: peer-memory inboxes for the partitioned exchange
 *   "p2p_force"      0        0..1      U: create the inbox on a one-rank communicator too
 *   "build_trace"    0        0..1      host timestamps of the build phases on stderr
 *   "remote_compact" 1        0..1      U: partitioned DI_ASYNC cycles through peer memory keep a
 *                                          compact accumulator for the hot targets of the other
 *                                          ranges and write pushes to colder remote targets as
 *                                          records straight into the owner's inbox (0: the
 *                                          global-size accumulator and its compaction scan)
 *   "remote_tier"    0        >= 0      U: hot remote targets per range (0: half the L2 over G)
 *   "long_lanes"     1        0..1      U: DI_ASYNC long rows (> 256 links) with lane-consecutive
 *                                          targets (0: int4 groups per lane)
 *   "row_sort"       0        0..1      U: one-GPU build without DI_DEDUP / DI_DROP_SELF_LOOPS /
 *                                          DI_BUILD_CSC by a counting sort on sources and a
 *                                          segmented sort of the rows (0: 64-bit key radix sort)
 *   "line_spread"    16       1,2,4,8,16 U: nodes of one rank class per 16-node L2 line of the
 *                                          relabelling (16: hot nodes packed; smaller spreads the
 *                                          hot set over more lines)
 *   "warm"           -1       -1..65536 U: warm tier of DI_ASYNC on one GPU, skewed graphs with
 *                                          n >= 8 x (warm + 64): the `warm` ranks after the 64 hot
 *                                          ones are placed one every 2^warm_shift ids, and every CTA
 *                                          of the cycle kernel accumulates its pushes to them and to
 *                                          the hot ids in shared memory (as many as fit without
 *                                          lowering occupancy), flushed into F when the CTA leaves
 *                                          the cycle (-1: as many as fit, 4032 on B200; 0: off)
 *   "warm_flush"     0        >= 0      U: the cycle kernel's CTAs also flush the warm tier into F
 *                                          every k of their tiles (0: only when they leave the cycle)
 *   "dist_parts"     1        1..64     U: partitioned DI_ASYNC solves run each rank's cycle in k
 *                                          parts of its tiles, every part followed by the exchange
 *                                          (remote fluid arrives within the cycle; the threshold
 *                                          r/L is taken per part; di_stats.sweeps counts parts)
 *   "warm_shift"     0        0..30     U: warm ranks one every 2^k ids (0: auto, the warm ids
 *                                          spanning about the first eighth of the range or of the
 *                                          first tier)
 * DI_EINVAL for an unknown name or a value out of range (integers must be integral). */
di_status di_set_option(const char *name, double value);
di_status di_get_option(const char *name, double *value);

/* DI-SOP threshold scale: later solves select F_i > alpha * (r/L) * #out_i.
 * alpha = 1 (the default) is the paper's rule and computes bit for bit the same
 * threshold; alpha > 1 diffuses fewer, larger amounts. alpha must be finite and > 0 (DI_EINVAL).
 * On a partitioned graph every rank must set the same value. */
di_status di_set_threshold_scale(di_graph g, double alpha);

/* Move the handle to another stream (cudaStream_t; NULL = legacy default stream): waits for the
 * work enqueued on the current stream, then every later call of this handle enqueues on `stream`
 * (e.g. upload on a low-priority stream while another graph solves, then solve on a high-priority
 * one). Not thread-safe with other calls on the same handle. */
di_status di_graph_set_stream(di_graph g, void *stream);

/* Node slice [lo, hi) owned by this rank ([0, n) on one GPU). */
di_status di_graph_range(di_graph g, int64_t *lo, int64_t *hi);

/* Number of links kept after DI_DEDUP / DI_DROP_SELF_LOOPS (this rank's links on multi-GPU). */
di_status di_graph_links(di_graph g, int64_t *n_links);

/* Solve X = P.X + B (§1) by D-iteration sweeps until ||F||_1 <= tol (BASELINE
 * north_star; or the paper's error with DI_PAPER_ERROR), or max_sweeps.
 *  d  : damping in (0, 1) (PAPER.md leaves it unstated: reading G1).
 *  B  : NULL -> uniform (1 - d)/N; else device pointer to this rank's slice, B >= 0.
 *  v  : DI_SOP / DI_CYC (the hot path) or a comparator (DI_PI_PULL, DI_PI_PUSH, DI_GS_BLOCK;
 *       for those tol bounds the scheme's own error estimate, P:176-180 / P:237-245, and
 *       di_history returns their x: normalised for PI, raw for GS).
 *  st : host pointer, filled on return (may be NULL).
 * Partitioned graph: collective; DI_SOP / DI_CYC with bulk push sweeps or DI_ASYNC cycles; B is this rank's slice
 * [lo, hi) in the caller's numbering; the stats are global (identical on every rank).
 * Returns DI_OK, DI_NOT_CONVERGED (state kept; DI_RESUME continues), or an error. */
di_status di_solve(di_graph g, double d, const double *B, double tol, di_variant v,
                   int64_t max_sweeps, uint32_t flags, di_stats *st);

/* ||F||_1 of the current state (exact deterministic tree sum) into *l1_out (host); if F_out
 * is not NULL, also copy this rank's F slice into it (device pointer). Collective on a
 * partitioned graph (the global sum). */
di_status di_residual(di_graph g, double *l1_out, double *F_out);

/* Copy this rank's history H (raw estimate of X) into H_out (device pointer). */
di_status di_history(di_graph g, double *H_out);

/* Per-sweep log of the last DI_TRACE solve (SPEC S:157 error_history): r_n (sum F at sweep
 * start as used by the threshold), |S_n|, links(S_n), mode (0 push, 1 pull). Host arrays of
 * capacity cap (any may be NULL); *n_out = sweeps logged (<= cap). */
di_status di_sweep_log(di_graph g, double *r, int64_t *selected, int64_t *links, uint8_t *mode,
                       int64_t cap, int64_t *n_out);

di_status di_graph_free(di_graph g);
const char *di_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DI_H */
