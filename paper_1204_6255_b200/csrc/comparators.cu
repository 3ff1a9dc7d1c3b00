// comparators.cu — GPU comparators of the paper (PI, PI', GS).
#include "di_common.cuh"

namespace di {

di_status run_comparator(Graph &g, double d, double tol, int variant, int64_t max_sweeps,
                         uint32_t flags, di_stats *st) {
  (void)g; (void)d; (void)tol; (void)variant; (void)max_sweeps; (void)flags; (void)st;
  set_error("di_solve: comparator variants are not available in this build");
  return DI_EINVAL;
}

}  // namespace di
