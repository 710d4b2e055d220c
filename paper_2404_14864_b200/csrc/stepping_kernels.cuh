// Time-stepping right-hand sides (timestepping.py), element-wise over either
// the (M+1)^2 grid (with the interior mask) or the n_ctl control points (no
// mask).  Each kernel folds in the blow-up norm max|u| of
// StepContext.check_stable (timestepping.py:172-175).
//
// Exterior nodes: every state field the steppers carry (u, F, F_prev, the
// Strang carry) is zero outside the mask — the startups build them from
// interior_field (timestepping.py:203-209, 243-274, 366-368) and every step
// masks what it returns — so at a masked-off node the recurrences give exactly
// 0 from zero inputs.  The kernels load the mask first and skip the field
// loads (and the Newton solve) there: only the zero stores remain (the
// exterior is 65-82 % of the grid in the bench geometries).
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

// Element-wise passes over n values, two adjacent elements per step (16-byte
// loads, aligned buffers: every field here is a whole torch allocation) and
// two steps in flight per thread; the odd tail element is done by thread 0.
// VEC = false is the scalar fallback for unaligned views.
template <bool VEC, typename F>
KFBI_DEV void elementwise_pairs(long n, F &&f) {
  const long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  if (VEC) {
    const long np = n >> 1;
    long i = tid;
    for (; i + stride < np; i += 2 * stride) f.template pair<2>(i, i + stride);
    if (i < np) f.template pair<1>(i, i);
    if (tid == 0 && (n & 1)) f.one(n - 1);
  } else {
    for (long i = tid; i < n; i += stride) f.one(i);
  }
}

// u <- mask ? u : 0 ; norm = max|u|   (np.where(ctx.mask, sol.u, 0.0))
template <typename T>
struct MaskNormOp {
  const unsigned char *__restrict__ mask;
  T *__restrict__ u;
  double mag;
  template <int K>
  KFBI_DEV void pair(long i0, long i1) {
    const long ii[2] = {i0, i1};
    T v[K][2];
    uchar2 mk[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      mk[k] = mask ? reinterpret_cast<const uchar2 *>(mask)[ii[k]] : make_uchar2(1, 1);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k][0] = v[k][1] = Sc<T>::zero();
      if (mk[k].x | mk[k].y) {                   // exterior pairs: zero stores only
        if constexpr (std::is_same<T, double>::value) {
          const double2 w = reinterpret_cast<const double2 *>(u)[ii[k]];
          v[k][0] = w.x;
          v[k][1] = w.y;
        } else {                                 // complex: one 16-byte load per element
          if (mk[k].x) v[k][0] = u[2 * ii[k]];
          if (mk[k].y) v[k][1] = u[2 * ii[k] + 1];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!mk[k].x) { v[k][0] = Sc<T>::zero(); u[2 * ii[k]] = v[k][0]; }
      if (!mk[k].y) { v[k][1] = Sc<T>::zero(); u[2 * ii[k] + 1] = v[k][1]; }
      mag = nanmax(mag, nanmax(Sc<T>::abs(v[k][0]), Sc<T>::abs(v[k][1])));
    }
  }
  KFBI_DEV void one(long i) {
    const bool in = !mask || mask[i];           // (exterior values are not read)
    T v = in ? u[i] : Sc<T>::zero();
    if (!in) u[i] = v;
    mag = nanmax(mag, Sc<T>::abs(v));
  }
};

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) mask_norm_kernel(long n, const unsigned char *mask, T *u,
                                                        unsigned long long *norm) {
  MaskNormOp<T> op{mask, u, 0.0};
  elementwise_pairs<VEC>(n, op);
  block_nanmax_to(norm, op.mag);
}

// heat (timestepping.py:218-228): u <- mask u;  F_new = a u - F_old
struct HeatOp {
  const unsigned char *__restrict__ mask;
  double *__restrict__ u;
  const double *__restrict__ F_old;
  double *__restrict__ F_new;
  double a, mag;
  bool ext_zero;                  // F_new is already zero outside the mask
  template <int K>
  KFBI_DEV void pair(long i0, long i1) {
    const long ii[2] = {i0, i1};
    double2 v[K], fo[K];
    uchar2 mk[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      mk[k] = mask ? reinterpret_cast<const uchar2 *>(mask)[ii[k]] : make_uchar2(1, 1);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k] = fo[k] = make_double2(0.0, 0.0);
      if (mk[k].x | mk[k].y) {
        v[k] = reinterpret_cast<const double2 *>(u)[ii[k]];
        fo[k] = reinterpret_cast<const double2 *>(F_old)[ii[k]];
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!mk[k].x || !mk[k].y) {
        if (!mk[k].x) v[k].x = 0.0;
        if (!mk[k].y) v[k].y = 0.0;
        reinterpret_cast<double2 *>(u)[ii[k]] = v[k];
      }
      if (!ext_zero || (mk[k].x | mk[k].y))
        reinterpret_cast<double2 *>(F_new)[ii[k]] = make_double2(a * v[k].x - fo[k].x, a * v[k].y - fo[k].y);
      mag = nanmax(mag, nanmax(fabs(v[k].x), fabs(v[k].y)));
    }
  }
  KFBI_DEV void one(long i) {
    const bool in = !mask || mask[i];
    const double v = in ? u[i] : 0.0;
    if (!in) u[i] = v;
    F_new[i] = a * v - F_old[i];
    mag = nanmax(mag, fabs(v));
  }
};

template <bool VEC>
__global__ void __launch_bounds__(256) heat_rhs_kernel(long n, const unsigned char *mask, double *u,
                                                       const double *F_old, double *F_new, double a,
                                                       unsigned long long *norm, bool ext_zero) {
  HeatOp op{mask, u, F_old, F_new, a, 0.0, ext_zero && mask != nullptr};
  elementwise_pairs<VEC>(n, op);
  block_nanmax_to(norm, op.mag);
}

// wave (timestepping.py:284-297)
//   un <- mask un;  F_new = (2 un - uc) kw + coef (kw un - fc) + (kw uc - fp)
struct WaveOp {
  const unsigned char *__restrict__ mask;
  double *__restrict__ un;
  const double *__restrict__ uc, *__restrict__ fc, *__restrict__ fp;
  double *__restrict__ F_new;
  double kw, coef, mag;
  bool ext_zero;                  // F_new is already zero outside the mask
  KFBI_DEV double f(double v, double c, double fcv, double fpv) const {
    return (2.0 * v - c) * kw + coef * (kw * v - fcv) + (kw * c - fpv);
  }
  template <int K>
  KFBI_DEV void pair(long i0, long i1) {
    const long ii[2] = {i0, i1};
    double2 v[K], c[K], a[K], b[K];
    uchar2 mk[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      mk[k] = mask ? reinterpret_cast<const uchar2 *>(mask)[ii[k]] : make_uchar2(1, 1);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k] = c[k] = a[k] = b[k] = make_double2(0.0, 0.0);
      if (mk[k].x | mk[k].y) {
        v[k] = reinterpret_cast<const double2 *>(un)[ii[k]];
        c[k] = reinterpret_cast<const double2 *>(uc)[ii[k]];
        a[k] = reinterpret_cast<const double2 *>(fc)[ii[k]];
        b[k] = reinterpret_cast<const double2 *>(fp)[ii[k]];
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!mk[k].x || !mk[k].y) {
        if (!mk[k].x) v[k].x = 0.0;
        if (!mk[k].y) v[k].y = 0.0;
        reinterpret_cast<double2 *>(un)[ii[k]] = v[k];
      }
      if (!ext_zero || (mk[k].x | mk[k].y))
        reinterpret_cast<double2 *>(F_new)[ii[k]] =
            make_double2(f(v[k].x, c[k].x, a[k].x, b[k].x), f(v[k].y, c[k].y, a[k].y, b[k].y));
      mag = nanmax(mag, nanmax(fabs(v[k].x), fabs(v[k].y)));
    }
  }
  KFBI_DEV void one(long i) {
    const bool in = !mask || mask[i];
    const double v = in ? un[i] : 0.0;
    if (!in) un[i] = v;
    F_new[i] = f(v, uc[i], fc[i], fp[i]);
    mag = nanmax(mag, fabs(v));
  }
};

template <bool VEC>
__global__ void __launch_bounds__(256) wave_rhs_kernel(long n, const unsigned char *mask, double *un,
                                                       const double *uc, const double *fc,
                                                       const double *fp, double *F_new, double kw,
                                                       double coef, unsigned long long *norm,
                                                       bool ext_zero) {
  WaveOp op{mask, un, uc, fc, fp, F_new, kw, coef, 0.0, ext_zero && mask != nullptr};
  elementwise_pairs<VEC>(n, op);
  block_nanmax_to(norm, op.mag);
}

// u* of the Strang step (timestepping.py:410-418):
//   mode 0: u - (0.5 i tau) other   (first step, other = lap u0)
//   mode 1: 2 u - other             (other = u** of the previous step)
KFBI_DEV double2 ustar_of(int mode, double2 a, double2 b, double tau) {
  if (mode == 0) return csub(a, cmul(make_double2(0.0, 0.5 * tau), b));
  return csub(make_double2(2.0 * a.x, 2.0 * a.y), b);
}

__global__ void schr_ustar_kernel(long n, int mode, const double2 *__restrict__ u,
                                  const double2 *__restrict__ other, double tau,
                                  double2 *__restrict__ out) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    out[i] = ustar_of(mode, u[i], other[i], tau);
}

// dst[i] = src[idx[i]] (packing the interior nodes of a masked field for a
// compact device -> host copy of a step's result)
template <typename T>
__global__ void __launch_bounds__(256) gather_kernel(long n, const int *__restrict__ idx,
                                                     const T *__restrict__ src, T *__restrict__ dst) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
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
// With `other` != nullptr, u* is formed inline from (ustar = u, other, mode)
// (the schr_ustar_kernel expression), saving a full-grid write and read.
__global__ void __launch_bounds__(256)
nonlinear_phase_kernel(long n, const double2 *__restrict__ ustar, const double2 *__restrict__ other,
                       int mode, double tau, const double *__restrict__ v, double w, double c,
                       const unsigned char *__restrict__ mask, double2 *__restrict__ out,
                       double kre, double kim, double2 *__restrict__ F,
                       unsigned long long *max_res, bool ext_zero = false) {
  double worst = 0.0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) {                      // u* = 0 there: Newton returns 0, residual 0
      if (!ext_zero) {                           // (ext_zero: out / F already hold the zeros)
        out[i] = make_double2(0.0, 0.0);
        if (F) F[i] = make_double2(0.0, 0.0);
      }
      continue;
    }
    double r;
    const double2 us = other ? ustar_of(mode, ustar[i], other[i], tau) : ustar[i];
    double2 z = newton_node(us, v[i], w, c, r);
    worst = nanmax(worst, r);
    if (mask && !mask[i]) z = make_double2(0.0, 0.0);
    out[i] = z;
    if (F) F[i] = cmul(make_double2(kre, kim), z);
  }
  block_nanmax_to(max_res, worst);
}

// The same over an explicit list of the interior nodes (increasing flat
// indices) when the outputs' exterior is zero already
// (kfbi_plan_set_exterior_zero + kfbi_plan_set_interior_list): the Newton
// work is spread evenly over the threads instead of concentrating in the
// warps that cover the domain (the full-grid pass spent most of its time with
// exterior warps idle at the block reduction).
__global__ void __launch_bounds__(256)
nonlinear_phase_list_kernel(long n_int, const int *__restrict__ idx, const double2 *__restrict__ ustar,
                            const double2 *__restrict__ other, int mode, double tau,
                            const double *__restrict__ v, double w, double c,
                            double2 *__restrict__ out, double kre, double kim, double2 *__restrict__ F,
                            unsigned long long *max_res) {
  double worst = 0.0;
  const double2 kap = make_double2(kre, kim);
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n_int;
       q += (long)gridDim.x * blockDim.x) {
    const long i = idx[q];
    double r;
    const double2 us = other ? ustar_of(mode, ustar[i], other[i], tau) : ustar[i];
    const double2 z = newton_node(us, v[i], w, c, r);
    worst = nanmax(worst, r);
    out[i] = z;
    if (F) F[i] = cmul(kap, z);
  }
  block_nanmax_to(max_res, worst);
}

}  // namespace kfbi
