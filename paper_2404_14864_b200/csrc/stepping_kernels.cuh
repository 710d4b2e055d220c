// Time-stepping right-hand sides (timestepping.py), element-wise over either
// the (M+1)^2 grid (with the interior mask) or the n_ctl control points (no
// mask).  Each kernel folds in the blow-up norm max|u| of
// StepContext.check_stable (timestepping.py:172-175).
#pragma once

#include "common.cuh"

namespace kfbi {

KFBI_DEV void block_nanmax_to(unsigned long long *dst, double v) {
  __shared__ double red[32];
  v = warp_nanmax(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double x = lane < (blockDim.x >> 5) ? red[lane] : 0.0;
    x = warp_nanmax(x);
    if (lane == 0) atomic_max_nonneg(dst, x);
  }
}

// u <- mask ? u : 0 ; norm = max|u|   (np.where(ctx.mask, sol.u, 0.0))
template <typename T>
__global__ void mask_norm_kernel(long n, const unsigned char *mask, T *u,
                                 unsigned long long *norm) {
  double mag = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    T v = u[i];
    if (mask && !mask[i]) { v = Sc<T>::zero(); u[i] = v; }
    mag = nanmax(mag, Sc<T>::abs(v));
  }
  block_nanmax_to(norm, mag);
}

// heat (timestepping.py:218-228): u <- mask u;  F_new = a u - F_old
__global__ void heat_rhs_kernel(long n, const unsigned char *mask, double *u, const double *F_old,
                                double *F_new, double a, unsigned long long *norm) {
  double mag = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double v = u[i];
    if (mask && !mask[i]) { v = 0.0; u[i] = v; }
    F_new[i] = a * v - F_old[i];
    mag = nanmax(mag, fabs(v));
  }
  block_nanmax_to(norm, mag);
}

// wave (timestepping.py:284-297)
//   un <- mask un;  F_new = (2 un - uc) kw + coef (kw un - fc) + (kw uc - fp)
__global__ void wave_rhs_kernel(long n, const unsigned char *mask, double *un,
                                const double *uc, const double *fc, const double *fp,
                                double *F_new, double kw, double coef,
                                unsigned long long *norm) {
  double mag = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double v = un[i];
    if (mask && !mask[i]) { v = 0.0; un[i] = v; }
    const double c = uc[i];
    F_new[i] = (2.0 * v - c) * kw + coef * (kw * v - fc[i]) + (kw * c - fp[i]);
    mag = nanmax(mag, fabs(v));
  }
  block_nanmax_to(norm, mag);
}

// u* of the Strang step (timestepping.py:410-418):
//   mode 0: u - (0.5 i tau) other   (first step, other = lap u0)
//   mode 1: 2 u - other             (other = u** of the previous step)
__global__ void schr_ustar_kernel(long n, int mode, const double2 *u, const double2 *other,
                                  double tau, double2 *out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double2 a = u[i], b = other[i];
    if (mode == 0) out[i] = csub(a, cmul(make_double2(0.0, 0.5 * tau), b));
    else out[i] = csub(make_double2(2.0 * a.x, 2.0 * a.y), b);
  }
}

// Pointwise damped Newton of nonlinear_phase_step (timestepping.py:317-368)
// for u** + ic(v + w|u**|^2)u** = u* - ic(v + w|u*|^2)u*, c = tau/2.
// Per node this is exactly the reference's vectorised iteration: a node stops
// moving once its residual is <= tol, the step halves while the residual
// grows (at most 30 times), at most 50 Newton steps.
constexpr double NEWTON_TOL = 1e-12;
constexpr int NEWTON_MAX_ITER = 50;

KFBI_DEV double2 newton_node(double2 us, double v, double w, double c, double &res_out) {
  const double am = hypot(us.x, us.y);
  const double k0 = c * (v + w * (am * am));
  // rhs = u* - (i c nv) u*
  const double r1 = us.x - (0.0 * us.x - k0 * us.y);
  const double r2 = us.y - (0.0 * us.y + k0 * us.x);
  double a = us.x, b = us.y;
  auto resid = [&](double aa, double bb, double &g1, double &g2) {
    const double nv = v + w * (aa * aa + bb * bb);
    g1 = aa - c * nv * bb - r1;
    g2 = bb + c * nv * aa - r2;
  };
  double g1, g2;
  resid(a, b, g1, g2);
  double res = fmax(fabs(g1), fabs(g2));
  for (int it = 0; it < NEWTON_MAX_ITER; ++it) {
    if (!(res > NEWTON_TOL)) break;
    const double nv = v + w * (a * a + b * b);
    const double j11 = 1.0 - 2.0 * c * w * a * b;
    const double j12 = -c * nv - 2.0 * c * w * b * b;
    const double j21 = c * nv + 2.0 * c * w * a * a;
    const double j22 = 1.0 + 2.0 * c * w * a * b;
    const double det = j11 * j22 - j12 * j21;
    const double da = (j22 * g1 - j12 * g2) / det;
    const double db = (j11 * g2 - j21 * g1) / det;
    double step = 1.0, an = a, bn = b, rn = res;
    for (int hv = 0; hv < 30; ++hv) {
      an = a - step * da;
      bn = b - step * db;
      resid(an, bn, g1, g2);
      rn = fmax(fabs(g1), fabs(g2));
      if (!(rn > res)) break;
      step = 0.5 * step;
    }
    a = an;
    b = bn;
    res = rn;
  }
  res_out = res;
  return make_double2(a, b);
}

// out = masked Newton(u*); optionally F = kappa * out; reports max residual.
__global__ void nonlinear_phase_kernel(long n, const double2 *ustar, const double *v, double w,
                                       double c, const unsigned char *mask, double2 *out,
                                       double kre, double kim, double2 *F,
                                       unsigned long long *max_res) {
  double worst = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    double r;
    double2 z = newton_node(ustar[i], v[i], w, c, r);
    worst = nanmax(worst, r);
    if (mask && !mask[i]) z = make_double2(0.0, 0.0);
    out[i] = z;
    if (F) F[i] = cmul(make_double2(kre, kim), z);
  }
  block_nanmax_to(max_res, worst);
}

}  // namespace kfbi
