// Node classification on the device (grid.py:122-155 of the reference,
// `classify`): interior iff the curve's level function phi(x_i, y_j) <=
// ON_CURVE_TOL.  The host arrays x, y are the grid coordinates bit for bit.
//
// Circle and ellipse levels are polynomials: evaluated with round-to-nearest
// intrinsics (no FMA contraction) they reproduce numpy's bits exactly.  The
// star level uses hypot / atan2 / cos, whose device and libm results may
// differ by a few ulp; nodes with |phi - tol| <= band (1e-12, far above the
// ~1e-14 worst-case discrepancy) are reported back and re-evaluated on the
// host with the reference formula, so the flags always equal the reference's.
#pragma once

#include "common.cuh"

namespace kfbi {

struct CurveDesc {
  int kind;                 // 0 circle, 1 ellipse, 2 star
  double cx, cy;
  double p0, p1, p2;        // circle: radius; ellipse: a, b; star: scale, c, lobes
};

KFBI_DEV double curve_level(const CurveDesc &c, double x, double y) {
  const double dx = __dsub_rn(x, c.cx), dy = __dsub_rn(y, c.cy);
  if (c.kind == 0) {                              // dx*dx + dy*dy - r**2
    return __dsub_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(c.p0, c.p0));
  }
  if (c.kind == 1) {                              // u*u + v*v - 1, u = dx / a
    const double u = __ddiv_rn(dx, c.p0), v = __ddiv_rn(dy, c.p1);
    return __dsub_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), 1.0);
  }
  // hypot(dx, dy) - s ((1 - c) + c cos(k atan2(dy, dx)))
  const double t = atan2(dy, dx);
  const double r = __dmul_rn(c.p0, __dadd_rn(__dsub_rn(1.0, c.p1), __dmul_rn(c.p1, cos(__dmul_rn(c.p2, t)))));
  return __dsub_rn(hypot(dx, dy), r);
}

__global__ void __launch_bounds__(256) classify_kernel(CurveDesc c, const double *__restrict__ x,
                                                       const double *__restrict__ y, int m, double tol,
                                                       double band, unsigned char *interior, int *n_amb,
                                                       long long *amb, int cap) {
  const int n1 = m + 1;
  const long long total = (long long)n1 * n1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q / n1), i = (int)(q - (long long)j * n1);
    const double lv = curve_level(c, x[i], y[j]);
    interior[q] = lv <= tol ? 1 : 0;
    if (band > 0.0 && fabs(lv - tol) <= band) {
      const int s = atomicAdd(n_amb, 1);
      if (s < cap) amb[s] = q;
    }
  }
}

}  // namespace kfbi
