// Dirichlet-zero box-solve passes, f64 (boxsolve.py:46-94): its own
// translation unit so the kernel instantiations compile in parallel.
#include "box_launch.cuh"

kfbi_status box_dirichlet_f64(kfbi_plan *p, int logm, bool tri, const kfbi::BoxArgs &a,
                              const void *rhs, double sign, const kfbi::CorrArgs<double> &c,
                              void *u, cudaStream_t s, int passes) {
  return kfbi::box_passes_reg<false>(p, logm, tri, a, rhs, sign, c, u, s, passes);
}
