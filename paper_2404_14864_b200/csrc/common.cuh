// Shared device helpers for the KFBI B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

#define KFBI_DEV __device__ __forceinline__

// ---- complex (interleaved double2, same memory layout as complex128) ----
KFBI_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
KFBI_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
KFBI_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
KFBI_DEV double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
KFBI_DEV double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
KFBI_DEV double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }
// a / b, written as numpy does for moderate magnitudes (Smith's scaling is not
// needed: |denominators| here are >= O(1/h^2) or O(kappa)).
KFBI_DEV double2 cdiv(double2 a, double2 b) {
  double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

KFBI_DEV double rdiv(double a, double s) { return a / s; }
KFBI_DEV double2 rdiv(double2 a, double s) { return make_double2(a.x / s, a.y / s); }

// Scalar type traits for the f64 / c128 kernels.
template <typename T> struct Sc;
template <> struct Sc<double> {
  static KFBI_DEV double zero() { return 0.0; }
  static KFBI_DEV double one() { return 1.0; }
  static KFBI_DEV double abs(double v) { return fabs(v); }
  static KFBI_DEV double add(double a, double b) { return a + b; }
  static KFBI_DEV double sub(double a, double b) { return a - b; }
  static KFBI_DEV double mul(double a, double b) { return a * b; }
  static KFBI_DEV double rmul(double a, double s) { return a * s; }
  // kappa is real on the f64 path
  static KFBI_DEV double kmul(double kre, double /*kim*/, double a) { return kre * a; }
};
template <> struct Sc<double2> {
  static KFBI_DEV double2 zero() { return make_double2(0.0, 0.0); }
  static KFBI_DEV double2 one() { return make_double2(1.0, 0.0); }
  static KFBI_DEV double abs(double2 v) { return hypot(v.x, v.y); }
  static KFBI_DEV double2 add(double2 a, double2 b) { return cadd(a, b); }
  static KFBI_DEV double2 sub(double2 a, double2 b) { return csub(a, b); }
  static KFBI_DEV double2 mul(double2 a, double2 b) { return cmul(a, b); }
  static KFBI_DEV double2 rmul(double2 a, double s) { return cscale(a, s); }
  static KFBI_DEV double2 kmul(double kre, double kim, double2 a) {
    return cmul(make_double2(kre, kim), a);
  }
};

// Non-negative doubles order like their bit patterns (NaN above +inf), so a
// 64-bit integer atomicMax is an exact, order-independent max reduction.
KFBI_DEV void atomic_max_nonneg(unsigned long long *addr, double v) {
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

KFBI_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// fmax drops NaN; the residual reduction must propagate it like np.max.
KFBI_DEV double nanmax(double a, double b) { return (a != a || a > b) ? a : b; }

KFBI_DEV double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

KFBI_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
