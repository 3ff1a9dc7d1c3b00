/* oracle/di_oracle.c — plain, slow, single-threaded CPU oracle for the D-iteration hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The product
 * path (paper_1204_6255_b200/) never links, imports or executes it, and this file
 * shares no code, header, helper or constant with the CUDA path.
 *
 * Source of truth: /root/reference/PAPER.md (cited "P:<line>", section in brackets).
 * Every loop below is the paper's pseudo-code (§2.5) written
 * out in C, in the paper's order and notation, in IEEE fp64 with no FMA
 * contraction (build with -O2 -ffp-contract=off). Where the paper is garbled or
 * silent the reading taken is the one listed in DESIGN.md §"Readings" (G1..G22,
 * after SURVEY.md §8(c)); each use is marked "[Gn]".
 *
 * Parity pins (tests/test_oracle.py): exact rationals of tests/golden/pins.txt
 * (hand-derived), a dense solve of (I-P)X = B for N <= 64,
 * scipy.sparse spsolve at C1, the invariants F = B + P.H - H and
 * ||X - H||_1 <= ||F||_1/(1-d), Neumann partial sums for bulk DI-CYC, closure
 * drainage, and the starvation guard cases. Every function here is pinned.
 *
 * Graph input: a link list (src[k] -> dst[k]), k in [0, L). P_ji = d/#out_i per
 * link i->j, duplicates counted (vector semantics), self-loops folded
 * (P:259-263). Adjacency is rebuilt here as the paper's l_out / l_in vectors
 * (P:67-71): link order within each vector is the link-list order.
 */
#include <math.h>
#include <stdint.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t cycles;            /* outer while-loop iterations ("cycles")                */
  int64_t diffusions;        /* link diffusions: sum of out[i] over diffused nodes [G12]     */
  int64_t guard_sweeps;      /* starvation-guard DI-CYC sweeps [G5]                          */
  int64_t selected;          /* total nodes diffused                                         */
  int64_t converged;         /* 1 if the stop test passed                                    */
  double residual;           /* sum F at exit (DI) / last error estimate (PI, PI', GS)       */
  double e;                  /* dangling absorbed mass                        */
  double eq_iter;            /* diffusions / L [G12]                                         */
  double solve_seconds;      /* wall time of the iteration loop only (adjacency build excluded,
                                as the paper times "Init" separately)                */
} orc_stats;

static double now_seconds(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* ------------------------------------------------------------------ adjacency */
typedef struct {
  int64_t n, l;
  int64_t *out_ptr; int32_t *out_idx;   /* l_out[i]: iterator for column i */
  int64_t *in_ptr;  int32_t *in_idx;    /* l_in[i]:  iterator for row i    */
  int32_t *out;                         /* out[i]: out-degree              */
  int32_t *loop;                        /* number of self-loop copies of i [G6]    */
} orc_graph;

static void g_free(orc_graph *g) {
  free(g->out_ptr); free(g->out_idx); free(g->in_ptr); free(g->in_idx); free(g->out); free(g->loop);
}
static int g_build(orc_graph *g, const int32_t *src, const int32_t *dst, int64_t L, int64_t N, int need_in) {
  memset(g, 0, sizeof *g);
  g->n = N; g->l = L;
  g->out_ptr = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
  g->out_idx = (int32_t *)malloc((size_t)(L > 0 ? L : 1) * sizeof(int32_t));
  g->out = (int32_t *)calloc((size_t)N, sizeof(int32_t));
  g->loop = (int32_t *)calloc((size_t)N, sizeof(int32_t));
  if (!g->out_ptr || !g->out_idx || !g->out || !g->loop) return -1;
  for (int64_t k = 0; k < L; k++) {
    if (src[k] < 0 || src[k] >= N || dst[k] < 0 || dst[k] >= N) return -1;
    g->out[src[k]]++;
    if (src[k] == dst[k]) g->loop[src[k]]++;
  }
  for (int64_t i = 0; i < N; i++) g->out_ptr[i + 1] = g->out_ptr[i] + g->out[i];
  int64_t *cur = (int64_t *)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < N; i++) cur[i] = g->out_ptr[i];
  for (int64_t k = 0; k < L; k++) g->out_idx[cur[src[k]]++] = dst[k];   /* push_back in file order */
  if (need_in) {
    int64_t *cnt = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
    for (int64_t k = 0; k < L; k++) cnt[dst[k] + 1]++;
    for (int64_t i = 0; i < N; i++) cnt[i + 1] += cnt[i];
    g->in_ptr = cnt;
    g->in_idx = (int32_t *)malloc((size_t)(L > 0 ? L : 1) * sizeof(int32_t));
    for (int64_t i = 0; i < N; i++) cur[i] = g->in_ptr[i];
    for (int64_t k = 0; k < L; k++) g->in_idx[cur[dst[k]]++] = src[k];
  }
  free(cur);
  return 0;
}

static int bad_args(int64_t L, int64_t N, double d) {
  return N < 1 || L < 0 || !(d > 0.0 && d < 1.0);
}

/* ===================================================================== D-iteration
 * §2.5.4 DI-CYC and §2.5.5 DI-SOP.
 *
 *   hist = 0; fluid = (1-d)/N; e = 0
 *   while error > target:
 *     [SOP: r = sum fluid, once per cycle, G3]
 *     for i in 0..N-1 (ascending, live fluid) [G13]:
 *       if fluid[i] > 0            (DI-CYC)
 *       if fluid[i] > r/L*out[i]   (DI-SOP, literal order [G4])
 *         transit = loop ? fluid*out/(out - k*d) : fluid                  ([G6])
 *         hist[i] += transit; fluid[i] = 0
 *         if out[i] == 0: e += transit                                    ([G2])
 *         else: sent = transit*d/out[i]; fluid[j] += sent, j in l_out[i], j != i   ([G7])
 *     error = sum fluid / (1 - d - d*e)
 *
 * Stop test [G9, G21]: before each cycle, r = sum fluid (ascending order [G14]);
 * stop_mode 0 (default, BASELINE north_star): r <= tol;
 * stop_mode 1 (paper): r/(1-d-d*e) <= tol.
 * Starvation guard [G5, SPEC S:247]: if a DI-SOP cycle diffuses no node while the stop
 * test fails, one DI-CYC cycle is run.
 */
static int64_t di_cycle(const orc_graph *g, double *F, double *H, double *e, double d,
                        int sop, double t, int64_t *diff, int64_t *sel) {
  int64_t selected = 0;
  for (int64_t i = 0; i < g->n; i++) {
    double thr = sop ? t * (double)g->out[i] : 0.0;
    if (F[i] > thr) {
      double transit;
      if (g->loop[i] > 0)
        transit = F[i] * (double)g->out[i] / ((double)g->out[i] - (double)g->loop[i] * d);
      else
        transit = F[i];
      H[i] += transit;
      F[i] = 0.0;
      selected++;
      if (g->out[i] == 0) {
        *e += transit;
      } else {
        double sent = transit * d / (double)g->out[i];
        for (int64_t k = g->out_ptr[i]; k < g->out_ptr[i + 1]; k++) {
          int32_t j = g->out_idx[k];
          if (j != i) F[j] += sent;
        }
        *diff += g->out[i];
      }
    }
  }
  *sel += selected;
  return selected;
}

static double sum_seq(const double *x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; i++) s += x[i];
  return s;
}

/* Sequential D-iteration. B = NULL -> uniform (1-d)/N. H_out, F_out: N doubles.
 * r_hist (nullable, cap entries): r at the start of every cycle. Returns 0 converged,
 * 1 not converged (max_cycles), -1 invalid arguments. */
int orc_di(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d,
           const double *B, double tol, int sop, int64_t max_cycles, int stop_mode,
           double *H_out, double *F_out, orc_stats *st, double *r_hist, int64_t hist_cap) {
  memset(st, 0, sizeof *st);
  if (bad_args(L, N, d) || !(tol > 0.0)) return -1;
  orc_graph g;
  if (g_build(&g, src, dst, L, N, 0)) { g_free(&g); return -1; }
  double *F = F_out, *H = H_out, e = 0.0;
  for (int64_t i = 0; i < N; i++) { H[i] = 0.0; F[i] = B ? B[i] : (1 - d) / N; }
  int64_t diff = 0, sel = 0;
  int rc = 1;
  double t_start = now_seconds();
  for (;;) {
    double r = sum_seq(F, N);
    if (r_hist && st->cycles < hist_cap) r_hist[st->cycles] = r;
    double err = stop_mode ? r / (1 - d - d * e) : r;
    st->residual = r;
    if (err <= tol) { rc = 0; break; }
    if (st->cycles >= max_cycles) break;
    double t = (L > 0) ? r / (double)L : 0.0;        /* r/L, once per cycle [G3, G4] */
    int64_t s = di_cycle(&g, F, H, &e, d, sop, t, &diff, &sel);
    if (s == 0) { di_cycle(&g, F, H, &e, d, 0, 0.0, &diff, &sel); st->guard_sweeps++; }
    st->cycles++;
  }
  st->solve_seconds = now_seconds() - t_start;
  st->converged = (rc == 0);
  st->diffusions = diff; st->selected = sel; st->e = e;
  st->eq_iter = L > 0 ? (double)diff / (double)L : 0.0;
  g_free(&g);
  return rc;
}

/* ============================================ bulk-synchronous sweep [DESIGN.md R1]
 * The GPU's reformulation of one D-iteration cycle (SURVEY §8(a) a3+a5): every node is
 * tested against the SNAPSHOT F_n (not the live F), all selected nodes move their fluid
 * into H, and only then is the fluid pushed. The per-node arithmetic is the paper's
 * (P:258-274). One call = one sweep; F, H, e are updated in place.
 * sel_T (nullable, N): transit of node i if selected, else 0; sel_mask (nullable, N): 1 if selected.
 * q_out / s_out (nullable): sum of unselected F and sum over selected non-dangling i of
 * transit*d*(out-k)/out (both ascending-order sums). Returns the number selected. */
static int64_t bulk_sweep_g(const orc_graph *gp, double d, double *F, double *H, double *e, int sop,
                            double r, double *sel_T, uint8_t *sel_mask, double *q_out, double *s_out,
                            int64_t *diffusions) {
  const orc_graph g = *gp;
  int64_t N = g.n, L = g.l;
  double t = (L > 0) ? r / (double)L : 0.0;
  double *T = (double *)calloc((size_t)N, sizeof(double));
  uint8_t *m = (uint8_t *)calloc((size_t)N, 1);
  int64_t count = 0, diff = 0;
  double q = 0.0, s = 0.0;
  for (int64_t i = 0; i < N; i++) {                 /* selection on the snapshot */
    double thr = sop ? t * (double)g.out[i] : 0.0;
    if (F[i] > thr) {
      m[i] = 1; count++;
      if (g.loop[i] > 0)
        T[i] = F[i] * (double)g.out[i] / ((double)g.out[i] - (double)g.loop[i] * d);
      else
        T[i] = F[i];
      H[i] += T[i];
      F[i] = 0.0;
      if (g.out[i] == 0) *e += T[i];
      else s += T[i] * d * ((double)g.out[i] - (double)g.loop[i]) / (double)g.out[i];
    } else {
      q += F[i];
    }
  }
  for (int64_t i = 0; i < N; i++) {                 /* push */
    if (!m[i] || g.out[i] == 0) continue;
    double sent = T[i] * d / (double)g.out[i];
    for (int64_t k = g.out_ptr[i]; k < g.out_ptr[i + 1]; k++) {
      int32_t j = g.out_idx[k];
      if (j != i) F[j] += sent;
    }
    diff += g.out[i];
  }
  if (sel_T) memcpy(sel_T, T, (size_t)N * sizeof(double));
  if (sel_mask) memcpy(sel_mask, m, (size_t)N);
  if (q_out) *q_out = q;
  if (s_out) *s_out = s;
  if (diffusions) *diffusions += diff;
  free(T); free(m);
  return count;
}
int64_t orc_bulk_sweep(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d,
                       double *F, double *H, double *e, int sop, double r,
                       double *sel_T, uint8_t *sel_mask, double *q_out, double *s_out,
                       int64_t *diffusions) {
  orc_graph g;
  if (bad_args(L, N, d) || g_build(&g, src, dst, L, N, 0)) { g_free(&g); return -1; }
  int64_t c = bulk_sweep_g(&g, d, F, H, e, sop, r, sel_T, sel_mask, q_out, s_out, diffusions);
  g_free(&g);
  return c;
}

/* Bulk-synchronous D-iteration to convergence (same stop rule and guard as orc_di). */
int orc_bulk_di(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d,
                const double *B, double tol, int sop, int64_t max_cycles,
                double *H_out, double *F_out, orc_stats *st) {
  memset(st, 0, sizeof *st);
  if (bad_args(L, N, d) || !(tol > 0.0)) return -1;
  orc_graph g;
  if (g_build(&g, src, dst, L, N, 0)) { g_free(&g); return -1; }
  double *F = F_out, *H = H_out, e = 0.0;
  for (int64_t i = 0; i < N; i++) { H[i] = 0.0; F[i] = B ? B[i] : (1 - d) / N; }
  int64_t diff = 0;
  int rc = 1;
  for (;;) {
    double r = sum_seq(F, N);
    st->residual = r;
    if (r <= tol) { rc = 0; break; }
    if (st->cycles >= max_cycles) break;
    int64_t c = bulk_sweep_g(&g, d, F, H, &e, sop, r, NULL, NULL, NULL, NULL, &diff);
    if (c == 0) { bulk_sweep_g(&g, d, F, H, &e, 0, 0.0, NULL, NULL, NULL, NULL, &diff); st->guard_sweeps++; }
    st->selected += c;
    st->cycles++;
  }
  st->converged = (rc == 0);
  st->diffusions = diff; st->e = e;
  st->eq_iter = L > 0 ? (double)diff / (double)L : 0.0;
  g_free(&g);
  return rc;
}

/* ========================================================= PI and PI'
 *   x_old = 1/N
 *   while error > target [G21: error starts at +inf]:
 *     x_new = (1-d)/N
 *     PI : x_new[i] += d*x_old[j]/out[j],  j in l_in[i]
 *     PI': transit = d*x_old[i]/out[i]; x_new[j] += transit, j in l_out[i]
 *     error = sum x_new; x_new[i] += (1.0-error)/N
 *     error = sum |x_new - x_old| * d/(1-d)
 *     x_old <- x_new [G20]
 * PI' uses PI's stop rule [G10]. x_out: the final x_new (normalised PageRank vector).
 * Each sweep counts L link traversals. */
static int pi_common(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d,
                     double target, int64_t max_iter, int by_column, double *x_out, orc_stats *st,
                     double *err_hist, int64_t hist_cap) {
  memset(st, 0, sizeof *st);
  if (bad_args(L, N, d) || !(target > 0.0)) return -1;
  orc_graph g;
  if (g_build(&g, src, dst, L, N, !by_column)) { g_free(&g); return -1; }
  double *x_old = (double *)malloc((size_t)N * sizeof(double));
  double *x_new = (double *)malloc((size_t)N * sizeof(double));
  for (int64_t i = 0; i < N; i++) x_old[i] = 1.0 / N;
  double error = INFINITY;
  int rc = 1;
  while (error > target) {
    if (st->cycles >= max_iter) break;
    for (int64_t i = 0; i < N; i++) x_new[i] = (1 - d) / N;
    if (!by_column) {
      for (int64_t i = 0; i < N; i++)
        for (int64_t k = g.in_ptr[i]; k < g.in_ptr[i + 1]; k++) {
          int32_t j = g.in_idx[k];
          x_new[i] += d * x_old[j] / g.out[j];
        }
    } else {
      for (int64_t i = 0; i < N; i++) {
        if (g.out[i] == 0) continue;               /* l_out[i] is empty: nothing to add */
        double transit = d * x_old[i] / g.out[i];
        for (int64_t k = g.out_ptr[i]; k < g.out_ptr[i + 1]; k++) x_new[g.out_idx[k]] += transit;
      }
    }
    error = 0.0;
    for (int64_t i = 0; i < N; i++) error += x_new[i];
    for (int64_t i = 0; i < N; i++) x_new[i] += (1.0 - error) / N;
    error = 0.0;
    for (int64_t i = 0; i < N; i++) error += fabs(x_new[i] - x_old[i]);
    error *= d / (1 - d);
    if (err_hist && st->cycles < hist_cap) err_hist[st->cycles] = error;
    double *t = x_old; x_old = x_new; x_new = t;   /* [G20] */
    st->cycles++;
    st->diffusions += L;
  }
  if (error <= target) rc = 0;
  memcpy(x_out, x_old, (size_t)N * sizeof(double));
  st->converged = (rc == 0);
  st->residual = error;
  st->eq_iter = (double)st->cycles;
  free(x_old); free(x_new); g_free(&g);
  return rc;
}
int orc_pi(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d, double target,
           int64_t max_iter, double *x_out, orc_stats *st, double *err_hist, int64_t hist_cap) {
  return pi_common(src, dst, L, N, d, target, max_iter, 0, x_out, st, err_hist, hist_cap);
}
int orc_pi_col(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d, double target,
               int64_t max_iter, double *x_out, orc_stats *st, double *err_hist, int64_t hist_cap) {
  return pi_common(src, dst, L, N, d, target, max_iter, 1, x_out, st, err_hist, hist_cap);
}

/* ============================================================== GS
 *   x = (1-d)/N
 *   while error > target [G21]:
 *     error = 0
 *     for i ascending: previous = x[i]; x[i] = (1-d)/N; diag = 1
 *       for j in l_in[i]: j != i ? x[i] += d*x[j]/out[j] : diag -= d/out[i]
 *       x[i] /= diag; error += x[i] - previous
 *     e = sum_{out[i]==0} x[i]  [G11, G22]
 *     error = error*d/(1 - d - d*e)
 * x_out: raw x (substochastic fixed point [G8]). */
int orc_gs(const int32_t *src, const int32_t *dst, int64_t L, int64_t N, double d, double target,
           int64_t max_iter, double *x_out, orc_stats *st, double *err_hist, int64_t hist_cap) {
  memset(st, 0, sizeof *st);
  if (bad_args(L, N, d) || !(target > 0.0)) return -1;
  orc_graph g;
  if (g_build(&g, src, dst, L, N, 1)) { g_free(&g); return -1; }
  double *x = x_out;
  for (int64_t i = 0; i < N; i++) x[i] = (1 - d) / N;
  double error = INFINITY, e = 0.0;
  int rc = 1;
  while (error > target) {
    if (st->cycles >= max_iter) break;
    error = 0.0;
    for (int64_t i = 0; i < N; i++) {
      double previous = x[i];
      x[i] = (1 - d) / N;
      double diag = 1.0;
      for (int64_t k = g.in_ptr[i]; k < g.in_ptr[i + 1]; k++) {
        int32_t j = g.in_idx[k];
        if (j != i) x[i] += d * x[j] / g.out[j];
        else diag -= d / g.out[i];
      }
      x[i] /= diag;
      error += x[i] - previous;
    }
    e = 0.0;
    for (int64_t i = 0; i < N; i++)
      if (g.out[i] == 0) e += x[i];
    error = error * d / (1 - d - d * e);
    if (err_hist && st->cycles < hist_cap) err_hist[st->cycles] = error;
    st->cycles++;
    st->diffusions += L;
  }
  if (error <= target) rc = 0;
  st->converged = (rc == 0);
  st->residual = error; st->e = e;
  st->eq_iter = (double)st->cycles;
  g_free(&g);
  return rc;
}
