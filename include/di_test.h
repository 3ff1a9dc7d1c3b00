/* include/di_test.h — test-only exports of libdi.so (not part of the product ABI).
 * They expose internal steps so that tests can check them bit for bit.
 */
#ifndef DI_TEST_H
#define DI_TEST_H

#include "di.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Run only the select/compact step (SURVEY §8(a) a3+a4: P:258/P:298 test, P:259-267 update)
 * on a caller snapshot F_in, H_in (host, this rank's n entries) with a frozen threshold fluid r.
 * Outputs (host):
 *   ids/vals/chunk : frontier entries in bin order [T | G | W | C], ascending node id inside a
 *                    bin; C entries repeat the node once per kChunk-link chunk, chunk = index.
 *                    vals = T_i*d/#out_i. Capacity `cap` entries (DI_EINVAL if too small).
 *   bin_off[5]     : bin boundaries in the concatenated arrays.
 *   scal[3]        : q (sum unselected F), s (sum T*d*(#out-k)/#out), e (dangling transit).
 *   counts[2]      : |S| (selected, dangling included), links(S).
 *   F_out, H_out   : state after the step (host, n entries each).
 * Leaves the handle's F and H set to F_out and H_out. */
di_status di_test_select(di_graph g, const double *F_in, const double *H_in, double r, double d,
                         di_variant v, int32_t *ids, double *vals, int32_t *chunk, int64_t cap,
                         int64_t bin_off[5], double scal[3], int64_t counts[2], double *F_out,
                         double *H_out);

/* Run ONE asynchronous cycle of the bench's kernel (k_cycle, DI_ASYNC; SURVEY §8(a) a2-a6 fused)
 * in its record mode on a caller snapshot F_in, H_in (host, n entries, caller's numbering) with
 * the cycle's threshold fluid r: every node is tested against (r/L)*#out_i (DI_SOP) or 0
 * (DI_CYC) and its fluid taken and folded exactly as in the product kernel, in
 * the same launch configuration, but nothing is pushed: the kernel writes T_out[i] = T_i and
 * v_out[i] = T_i*d/#out_i (0 for dangling nodes) for the selected nodes and leaves both 0
 * elsewhere (T_i > 0 for every selected node). With no push nothing else changes F during the
 * cycle, so the result must equal the oracle's bulk sweep on the same snapshot bit for bit.
 * Outputs (host, caller's numbering; any may be NULL): T_out, v_out, F_out, H_out (n each);
 * scal[3] = q (r - sum of taken fluid), s (sum v*(#out - k)), e (dangling transit);
 * counts[2] = |S| (selected, dangling included), links(S). Single-GPU graphs (DI_EINVAL else).
 * Leaves the handle's F and H set to F_out and H_out. */
di_status di_test_cycle(di_graph g, const double *F_in, const double *H_in, double r, double d,
                        di_variant v, double *T_out, double *v_out, double scal[3],
                        int64_t counts[2], double *F_out, double *H_out);

/* Internal numbering: old_of[k] = caller id of internal node k (identity with DI_NO_REORDER). */
di_status di_test_perm(di_graph g, int32_t *old_of);

/* Copy the device CSR (and CSC if built), in the internal numbering, to host arrays
 * (each may be NULL). */
di_status di_test_csr(di_graph g, int64_t *row_ptr, int32_t *col, int32_t *deg, int32_t *kloop,
                      int64_t *csc_ptr, int32_t *csc_row);

/* Bin thresholds compiled into the library: out[0..3] = kBinT, kBinG, kBinW, kChunk. */
di_status di_test_bins(int32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
