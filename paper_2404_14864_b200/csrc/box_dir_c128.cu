// Dirichlet-zero box-solve passes, c128 (boxsolve.py:46-94): its own
// translation unit so the kernel instantiations compile in parallel.
#include "box_launch.cuh"

kfbi_status box_dirichlet_c128(kfbi_plan *p, int logm, bool tri, const kfbi::BoxArgs &a,
                              const void *rhs, double sign, const kfbi::CorrArgs<double2> &c,
                              void *u, cudaStream_t s, int passes) {
  return kfbi::box_passes_reg<true>(p, logm, tri, a, rhs, sign, c, u, s, passes);
}
