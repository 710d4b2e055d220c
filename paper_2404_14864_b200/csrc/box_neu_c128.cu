// Neumann-zero box-solve passes, c128 (boxsolve.py:61-63, DCT-I): its own
// translation unit so the kernel instantiations compile in parallel.
#include "box_launch.cuh"

kfbi_status box_neumann_c128(kfbi_plan *p, int logm, const kfbi::BoxArgs &a, const void *rhs,
                            double sign, const kfbi::CorrArgs<double2> &c, void *u, cudaStream_t s) {
  return kfbi::box_neu_switch<true>(p, logm, a, rhs, sign, c, u, s);
}
