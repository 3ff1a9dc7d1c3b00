/* digen/gen.c — seeded synthetic link-list generators (input plumbing only).
 *
 * This module holds NONE of the D-iteration arithmetic. It produces the link
 * lists (i -> j) that both the CPU oracle (oracle/) and the CUDA path
 * (paper_1204_6255_b200/) consume, so that the two sides see identical inputs.
 * The recipes stand in for the paper's missing datasets (uk-2007-05 prefixes,
 * PAPER.md §2.6; gr0.California, §2.8); they never
 * reproduce those datasets. The recipes are stated in DESIGN.md §"Input recipe".
 *
 * Every random draw is a counter-based hash of (seed, tag, index, sub-index),
 * so the output is independent of the thread count and of the machine.
 * Output: links sorted by (src, dst); self-loops dropped and duplicates
 * removed unless the caller asks for the raw candidate list.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>
#include <stdio.h>
#include <time.h>
static double now_s(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
#define VLOG(...) do { if (getenv("DIGEN_VERBOSE")) { fprintf(stderr, __VA_ARGS__); } } while (0)

/* ---------------------------------------------------------------- hashing */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t h4(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  return mix64(mix64(mix64(seed ^ (tag << 56)) ^ a) + b);
}
/* uniform in [0,1) with 53 random bits */
static inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

/* ------------------------------------------------- Feistel relabelling */
typedef struct { int half; uint64_t mask; uint64_t key; int64_t n; } perm_t;
static perm_t perm_make(int64_t n, uint64_t seed) {
  perm_t p; int s = 0; while ((1LL << s) < n) s++;
  p.half = (s + 1) / 2; if (p.half == 0) p.half = 1;
  p.mask = (1ULL << p.half) - 1; p.key = mix64(seed ^ 0x5045524dULL); p.n = n;
  return p;
}
static inline uint64_t feistel(const perm_t *p, uint64_t x) {
  uint64_t L = (x >> p->half) & p->mask, R = x & p->mask;
  for (int r = 0; r < 4; r++) {
    uint64_t t = L ^ (mix64(R ^ (p->key + (uint64_t)r * 0x9E37ULL)) & p->mask);
    L = R; R = t;
  }
  return (L << p->half) | R;
}
/* bijection on [0, n) by cycle-walking */
static inline int64_t perm_apply(const perm_t *p, int64_t x) {
  uint64_t y = (uint64_t)x;
  do { y = feistel(p, y); } while (y >= (uint64_t)p->n);
  return (int64_t)y;
}

/* --------------------------------------------------------- R-MAT draw */
typedef struct {
  int64_t n; int s; uint64_t seed;
  uint32_t A, AB, ABC;     /* integer quadrant thresholds round(a*2^32) ... */
} rmat_t;
static inline uint32_t thr32(double x) {
  double v = floor(x * 4294967296.0 + 0.5);
  if (v >= 4294967295.0) return 0xFFFFFFFFu;
  if (v <= 0) return 0;
  return (uint32_t)v;
}
/* one R-MAT candidate (tag-separated stream); returns 0 if rejected (>= n) */
static inline int rmat_draw(const rmat_t *R, uint64_t tag, uint64_t e, int64_t *src, int64_t *dst) {
  uint64_t s = 0, d = 0, h = 0;
  uint64_t base = mix64(mix64(R->seed ^ (tag << 56)) ^ e);   /* == h4(seed,tag,e,.) prefix */
  for (int l = 0; l < R->s; l++) {
    if ((l & 1) == 0) h = mix64(base + (uint64_t)(l >> 1));
    uint32_t u = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
    int rb, cb;
    if (u < R->A) { rb = 0; cb = 0; }
    else if (u < R->AB) { rb = 0; cb = 1; }
    else if (u < R->ABC) { rb = 1; cb = 0; }
    else { rb = 1; cb = 1; }
    s = (s << 1) | (uint64_t)rb; d = (d << 1) | (uint64_t)cb;
  }
  if (s >= (uint64_t)R->n || d >= (uint64_t)R->n) return 0;
  *src = (int64_t)s; *dst = (int64_t)d; return 1;
}

/* ------------------------------------------------------- result handle */
typedef struct {
  int64_t n, l;
  int32_t *src, *dst;
  int64_t m_candidates, m_kept_raw;
} gen_result;

int64_t digen_len(const void *h) { return ((const gen_result *)h)->l; }
int64_t digen_nodes(const void *h) { return ((const gen_result *)h)->n; }
int64_t digen_raw(const void *h) { return ((const gen_result *)h)->m_kept_raw; }
void digen_copy(const void *h, int32_t *src, int32_t *dst) {
  const gen_result *r = (const gen_result *)h;
  memcpy(src, r->src, (size_t)r->l * 4); memcpy(dst, r->dst, (size_t)r->l * 4);
}
void digen_free(void *h) {
  gen_result *r = (gen_result *)h; if (!r) return;
  free(r->src); free(r->dst); free(r);
}

/* ------------------------------------------------------ thread helpers */
static int nthreads_default(int nt) {
  if (nt > 0) return nt;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  if (c < 1) c = 1; if (c > 64) c = 64;
  return (int)c;
}
typedef void (*range_fn)(void *ctx, int tid, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int tid; int64_t lo, hi; } job_t;
static void *job_run(void *a) { job_t *j = (job_t *)a; j->fn(j->ctx, j->tid, j->lo, j->hi); return NULL; }
static void parallel_for(int nt, int64_t n, range_fn fn, void *ctx) {
  pthread_t th[64]; job_t jb[64];
  for (int t = 0; t < nt; t++) {
    jb[t].fn = fn; jb[t].ctx = ctx; jb[t].tid = t;
    jb[t].lo = n * t / nt; jb[t].hi = n * (t + 1) / nt;
    pthread_create(&th[t], NULL, job_run, &jb[t]);
  }
  for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
}

/* growable per-thread link buffer, packed (src << 32 | dst) */
typedef struct { uint64_t *v; int64_t n, cap; } vec_t;
static void vpush(vec_t *v, int64_t s, int64_t d) {
  if (v->n == v->cap) { v->cap = v->cap ? v->cap * 2 : 1 << 16; v->v = (uint64_t *)realloc(v->v, (size_t)v->cap * 8); }
  v->v[v->n++] = ((uint64_t)s << 32) | (uint64_t)(uint32_t)d;
}

/* ------------------------------- counting sort by src + row sort/dedup */
static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b; return (x > y) - (x < y);
}
static void row_sort(uint32_t *a, int64_t n) {
  if (n < 24) {
    for (int64_t i = 1; i < n; i++) { uint32_t k = a[i]; int64_t j = i - 1; while (j >= 0 && a[j] > k) { a[j + 1] = a[j]; j--; } a[j + 1] = k; }
  } else qsort(a, (size_t)n, 4, cmp_u32);
}
typedef struct { vec_t *bufs; int nb; int64_t *cnt; int64_t *cursor; uint32_t *col; int64_t n; int dedup, drop_self; int64_t *newdeg; } csr_ctx;
static void csr_count(void *c_, int tid, int64_t lo, int64_t hi) {
  csr_ctx *c = (csr_ctx *)c_; (void)lo; (void)hi;
  vec_t *b = &c->bufs[tid];
  for (int64_t k = 0; k < b->n; k++) __atomic_fetch_add(&c->cnt[b->v[k] >> 32], 1, __ATOMIC_RELAXED);
}
static void csr_scatter(void *c_, int tid, int64_t lo, int64_t hi) {
  csr_ctx *c = (csr_ctx *)c_; (void)lo; (void)hi;
  vec_t *b = &c->bufs[tid];
  for (int64_t k = 0; k < b->n; k++) {
    int64_t s = (int64_t)(b->v[k] >> 32);
    int64_t pos = __atomic_fetch_add(&c->cursor[s], 1, __ATOMIC_RELAXED);
    c->col[pos] = (uint32_t)(b->v[k] & 0xFFFFFFFFu);
  }
}
static void csr_rows(void *c_, int tid, int64_t lo, int64_t hi) {
  csr_ctx *c = (csr_ctx *)c_; (void)tid;
  for (int64_t i = lo; i < hi; i++) {
    int64_t b = c->cnt[i], e = c->cnt[i + 1];
    uint32_t *a = c->col + b; int64_t n = e - b;
    row_sort(a, n);
    int64_t w = 0;
    for (int64_t k = 0; k < n; k++) {
      if (c->drop_self && (int64_t)a[k] == i) continue;
      if (c->dedup && w > 0 && a[w - 1] == a[k]) continue;
      a[w++] = a[k];
    }
    c->newdeg[i] = w;
  }
}
typedef struct { int64_t *cnt, *newoff; uint32_t *col; int32_t *src, *dst; } cpy_ctx;
static void csr_emit(void *c_, int tid, int64_t lo, int64_t hi) {
  cpy_ctx *c = (cpy_ctx *)c_; (void)tid;
  for (int64_t i = lo; i < hi; i++) {
    int64_t o = c->newoff[i], n = c->newoff[i + 1] - o;
    for (int64_t k = 0; k < n; k++) { c->src[o + k] = (int32_t)i; c->dst[o + k] = (int32_t)c->col[c->cnt[i] + k]; }
  }
}
static gen_result *finish(vec_t *bufs, int nt, int64_t n, int dedup, int drop_self) {
  gen_result *r = (gen_result *)calloc(1, sizeof(gen_result));
  r->n = n;
  int64_t total = 0; for (int t = 0; t < nt; t++) total += bufs[t].n;
  r->m_kept_raw = total;
  csr_ctx c; memset(&c, 0, sizeof c);
  c.bufs = bufs; c.nb = nt; c.n = n; c.dedup = dedup; c.drop_self = drop_self;
  c.cnt = (int64_t *)calloc((size_t)n + 1, 8);
  c.cursor = (int64_t *)malloc(((size_t)n + 1) * 8);
  c.newdeg = (int64_t *)malloc(((size_t)n + 1) * 8);
  c.col = (uint32_t *)malloc((size_t)(total ? total : 1) * 4);
  double t0 = now_s();
  parallel_for(nt, n, csr_count, &c);
  VLOG("count %.2f\n", now_s() - t0);
  /* exclusive scan (serial) */
  int64_t acc = 0;
  for (int64_t i = 0; i < n; i++) { int64_t v = c.cnt[i]; c.cnt[i] = acc; c.cursor[i] = acc; acc += v; }
  c.cnt[n] = acc;
  VLOG("scan %.2f\n", now_s() - t0);
  parallel_for(nt, n, csr_scatter, &c);
  VLOG("scatter %.2f\n", now_s() - t0);
  for (int t = 0; t < nt; t++) { free(bufs[t].v); bufs[t].v = NULL; }
  parallel_for(nt, n, csr_rows, &c);
  VLOG("rows %.2f\n", now_s() - t0);
  int64_t *newoff = c.cursor; acc = 0;
  for (int64_t i = 0; i < n; i++) { newoff[i] = acc; acc += c.newdeg[i]; }
  newoff[n] = acc;
  r->l = acc;
  r->src = (int32_t *)malloc((size_t)(acc ? acc : 1) * 4);
  r->dst = (int32_t *)malloc((size_t)(acc ? acc : 1) * 4);
  cpy_ctx cc = {c.cnt, newoff, c.col, r->src, r->dst};
  parallel_for(nt, n, csr_emit, &cc);
  VLOG("emit %.2f\n", now_s() - t0);
  free(c.cnt); free(c.cursor); free(c.newdeg); free(c.col);
  return r;
}

/* ====================================================== R-MAT + repair
 * Recipe (after SURVEY §8(d)):
 *  1. m candidates e: R-MAT quadrant descent with 32-bit integer thresholds,
 *     reject src/dst >= n, relabel both ends by a seeded Feistel bijection.
 *  2. D* (dangling, "0 out-degree") = {i : u(seed,'D',i) < p_dangling};
 *     Z* (zero in-degree) = {i notin D* : u(seed,'Z',i) < p_zero_in/(1-p_dangling)};
 *     chain windows: window w of 8 consecutive ids is a chain window if
 *     u(seed,'C',w) < 8*chain_heads; its head 8w has no in-link and members
 *     8w+1..8w+len (len in {2,3,4}) receive exactly one in-link, from their
 *     predecessor: recursive zero in-degree chains.
 *  3. drop candidates whose src in D*, or whose dst in Z* or in a chain.
 *  4. every i notin D* gets one extra out-link to the dst of a fresh R-MAT
 *     candidate (retrying until the target is a legal receiver and != i), so
 *     that out-degree 0 <=> i in D*.
 *  5. if repair_in: every legal receiver j gets one extra in-link from the src
 *     of a fresh candidate (retry until the source notin D* and != j).
 *  6. sort by (src,dst), drop self-loops, dedup (unless raw).
 */
typedef struct {
  rmat_t R; perm_t P; int64_t n, m;
  double p_dang, p_zin_cond, p_chain_win; int repair_in;
  vec_t *bufs;
} rmat_ctx;

static inline int chain_info(const rmat_ctx *c, int64_t x, int *is_head, int *is_member) {
  /* returns 1 if x is inside a chain (head or member) */
  *is_head = 0; *is_member = 0;
  if (c->p_chain_win <= 0) return 0;
  int64_t w = x >> 3, off = x & 7;
  uint64_t h = h4(c->R.seed, 'C', (uint64_t)w, 0);
  if (u01(h) >= c->p_chain_win) return 0;
  int len = 2 + (int)((h >> 3) % 3);
  if ((w << 3) + len >= c->n) return 0;
  if (off == 0) { *is_head = 1; return 1; }
  if (off <= len) { *is_member = 1; return 1; }
  return 0;
}
static inline int is_dangling(const rmat_ctx *c, int64_t x) {
  int hd, mb; if (chain_info(c, x, &hd, &mb)) return 0;
  return u01(h4(c->R.seed, 'D', (uint64_t)x, 0)) < c->p_dang;
}
/* may x receive ordinary links? (not Z*, not in a chain) */
static inline int is_receiver(const rmat_ctx *c, int64_t x) {
  int hd, mb; if (chain_info(c, x, &hd, &mb)) return 0;
  if (u01(h4(c->R.seed, 'D', (uint64_t)x, 0)) < c->p_dang) return 1;   /* dangling nodes receive */
  return !(u01(h4(c->R.seed, 'Z', (uint64_t)x, 0)) < c->p_zin_cond);
}
static void rmat_cands(void *c_, int tid, int64_t lo, int64_t hi) {
  rmat_ctx *c = (rmat_ctx *)c_;
  vec_t *b = &c->bufs[tid];
  for (int64_t e = lo; e < hi; e++) {
    int64_t s, d;
    if (!rmat_draw(&c->R, 'R', (uint64_t)e, &s, &d)) continue;
    s = perm_apply(&c->P, s); d = perm_apply(&c->P, d);
    if (is_dangling(c, s)) continue;
    if (!is_receiver(c, d)) continue;
    vpush(b, s, d);
  }
}
static void rmat_repairs(void *c_, int tid, int64_t lo, int64_t hi) {
  rmat_ctx *c = (rmat_ctx *)c_;
  vec_t *b = &c->bufs[tid];
  for (int64_t i = lo; i < hi; i++) {
    int hd, mb;
    if (chain_info(c, i, &hd, &mb)) {
      if (mb) vpush(b, i - 1, i);   /* predecessor -> member: the only in-link */
    }
    if (!is_dangling(c, i)) {      /* step 4: guaranteed out-link */
      for (uint64_t t = 0; t < 4096; t++) {
        int64_t s, d;
        if (!rmat_draw(&c->R, 'O', ((uint64_t)i << 12) | t, &s, &d)) continue;
        d = perm_apply(&c->P, d);
        if (d == i || !is_receiver(c, d)) continue;
        vpush(b, i, d); break;
      }
    }
    if (c->repair_in && is_receiver(c, i)) {   /* step 5: guaranteed in-link */
      for (uint64_t t = 0; t < 4096; t++) {
        int64_t s, d;
        if (!rmat_draw(&c->R, 'I', ((uint64_t)i << 12) | t, &s, &d)) continue;
        s = perm_apply(&c->P, s);
        if (s == i || is_dangling(c, s)) continue;
        vpush(b, s, i); break;
      }
    }
  }
}

void *digen_rmat(int64_t n, int64_t m, double a, double b, double cc, uint64_t seed,
                 double p_dangling, double p_zero_in, double chain_heads, int repair,
                 int repair_in, int raw, int nthreads) {
  if (n < 1 || n > 2147483647LL || m < 0) return NULL;
  int nt = nthreads_default(nthreads);
  rmat_ctx c; memset(&c, 0, sizeof c);
  int s = 0; while ((1LL << s) < n) s++;
  c.R.n = n; c.R.s = s; c.R.seed = seed;
  c.R.A = thr32(a); c.R.AB = thr32(a + b); c.R.ABC = thr32(a + b + cc);
  c.P = perm_make(n, seed);
  c.n = n; c.m = m;
  c.p_dang = repair ? p_dangling : 0.0;
  c.p_zin_cond = (repair && p_dangling < 1.0) ? p_zero_in / (1.0 - p_dangling) : 0.0;
  c.p_chain_win = repair ? chain_heads * 8.0 : 0.0;
  c.repair_in = repair && repair_in;
  c.bufs = (vec_t *)calloc((size_t)nt, sizeof(vec_t));
  double t0 = now_s();
  parallel_for(nt, m, rmat_cands, &c);
  VLOG("cands %.2f nt=%d\n", now_s() - t0, nt);
  if (repair) {
    /* repairs go into extra per-thread buffers appended to the same vectors */
    parallel_for(nt, n, rmat_repairs, &c);
  }
  gen_result *r = finish(c.bufs, nt, n, !raw, !raw);
  r->m_candidates = m;
  free(c.bufs);
  return r;
}

/* ====================================================== host-block graph
 * Recipe (BASELINE.json configs[2]): nodes are laid
 * out in contiguous blocks ("hosts") of size uniform in [bmin, bmax]; a node is
 * dangling with probability p_dangling; otherwise its out-degree is geometric
 * on {1,2,...} with mean mean_out; each link goes with probability p_intra to a
 * uniform target of its own block (!= self) and otherwise to a global target of
 * power-law rank (density ~ x^-beta on [1,n+1), beta = 1/(alpha_in - 1)), relabelled by a
 * seeded Feistel bijection.
 */
typedef struct {
  int64_t n; uint64_t seed; double p_dang, mean_out, p_intra, zexp, zmax;
  int32_t *blo, *bhi; perm_t P; vec_t *bufs;
} hb_ctx;
static void hb_rows(void *c_, int tid, int64_t lo, int64_t hi) {
  hb_ctx *c = (hb_ctx *)c_;
  vec_t *b = &c->bufs[tid];
  double q = 1.0 - 1.0 / c->mean_out, lq = log(q);
  for (int64_t i = lo; i < hi; i++) {
    if (u01(h4(c->seed, 'D', (uint64_t)i, 0)) < c->p_dang) continue;
    double u = 1.0 - u01(h4(c->seed, 'K', (uint64_t)i, 0));    /* (0,1] */
    int64_t k = 1 + (int64_t)floor(log(u) / lq);
    if (k > 100000) k = 100000;
    int64_t bl = c->blo[i], bh = c->bhi[i];
    for (int64_t t = 0; t < k; t++) {
      uint64_t h = h4(c->seed, 'H', (uint64_t)i, (uint64_t)t);
      double ui = u01(h);
      int64_t j;
      if (ui < c->p_intra) {
        uint64_t h2 = mix64(h);
        j = bl + (int64_t)(h2 % (uint64_t)(bh - bl - 1));
        if (j >= i) j++;
      } else {
        /* continuous power law on [1, n+1) with density ~ x^-beta, rank = floor(x) - 1 */
        double uz = u01(mix64(h ^ 0xABCDEFULL));
        double x = pow(1.0 + uz * (c->zmax - 1.0), c->zexp);
        int64_t rank = (int64_t)floor(x) - 1;
        if (rank < 0) rank = 0;
        if (rank >= c->n) rank = c->n - 1;
        j = perm_apply(&c->P, rank);
      }
      vpush(b, i, j);
    }
  }
}
void *digen_hostblock(int64_t n, int64_t bmin, int64_t bmax, double p_dangling, double mean_out,
                      double p_intra, double alpha_in, uint64_t seed, int raw, int nthreads) {
  if (n < 2 || n > 2147483647LL || bmin < 2 || bmax < bmin) return NULL;
  int nt = nthreads_default(nthreads);
  hb_ctx c; memset(&c, 0, sizeof c);
  c.n = n; c.seed = seed; c.p_dang = p_dangling; c.mean_out = mean_out; c.p_intra = p_intra;
  double beta = 1.0 / (alpha_in - 1.0);
  c.zexp = 1.0 / (1.0 - beta);
  c.zmax = pow((double)n + 1.0, 1.0 - beta);
  c.P = perm_make(n, seed ^ 0x484F5354ULL);
  c.blo = (int32_t *)malloc((size_t)n * 4); c.bhi = (int32_t *)malloc((size_t)n * 4);
  int64_t x = 0, bidx = 0;
  while (x < n) {
    int64_t sz = bmin + (int64_t)(h4(seed, 'B', (uint64_t)bidx, 0) % (uint64_t)(bmax - bmin + 1));
    int64_t e = x + sz; if (e > n || n - e < bmin) e = n;
    for (int64_t i = x; i < e; i++) { c.blo[i] = (int32_t)x; c.bhi[i] = (int32_t)e; }
    x = e; bidx++;
  }
  c.bufs = (vec_t *)calloc((size_t)nt, sizeof(vec_t));
  parallel_for(nt, n, hb_rows, &c);
  gen_result *r = finish(c.bufs, nt, n, !raw, !raw);
  free(c.bufs); free(c.blo); free(c.bhi);
  return r;
}
