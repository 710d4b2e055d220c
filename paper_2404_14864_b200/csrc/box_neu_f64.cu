// Neumann-zero box-solve passes, f64 (boxsolve.py:61-63, DCT-I): its own
// translation unit so the kernel instantiations compile in parallel.
#include "box_launch.cuh"

kfbi_status box_neumann_f64(kfbi_plan *p, int logm, const kfbi::BoxArgs &a, const void *rhs,
                            double sign, const kfbi::CorrArgs<double> &c, void *u, cudaStream_t s) {
  return kfbi::box_neu_switch<false>(p, logm, a, rhs, sign, c, u, s);
}
