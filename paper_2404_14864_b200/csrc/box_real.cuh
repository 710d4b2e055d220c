// Dirichlet box solve of REAL data at the largest size (M = 2L = 16384):
// one real row or column per CTA, its DST-I of length M computed with ONE
// complex FFT of length L = M/2 (the register engine at LOGN - 1: a single
// 512-thread CTA, 128 KB of shared memory) instead of a two-CTA cluster over
// distributed shared memory for packed pairs.
//
//   y_j = sin(pi j / M)(x_j + x_{M-j}) + (x_j - x_{M-j}) / 2      (real, j < M)
//   z_q = y_2q + i y_2q+1,  Zc = FFT_L(z)
//   Y_k = (Zc_k + conj Zc_{L-k}) / 2 - (i / 2) W^k (Zc_k - conj Zc_{L-k}),
//         W = exp(-2 pi i / M)                       (real FFT of length M)
//   C_2k = -2 Im Y_k,  C_1 = Re Y_0,  C_2k+1 = C_2k-1 + 2 Re Y_k
//
// Shared memory holds x (and later C) as pairs: slot q = (x_2q, x_2q+1).
// Same panel layout and slab conventions as box_reg.cuh (four real spectral
// columns per panel strip), so the slab-decomposed solve uses these kernels
// unchanged.
#pragma once

#include "box_reg.cuh"

namespace kfbi {
namespace realdst {

// y pairs from the staged x pairs (x_0 = 0 in slot 0, x_M = 0 implicit)
template <int LOGL>
KFBI_DEV void pre(double2 (&v)[reg::E], const reg::View<LOGL> &sm, int t,
                  const double *__restrict__ sinv) {
  constexpr int L = 1 << LOGL;
  constexpr int T = reg::Cfg<LOGL>::T;
#pragma unroll
  for (int m = 0; m < reg::E; ++m) {
    const int q = t + m * T;
    const double2 a = sm[q];                           // x_2q, x_2q+1
    const double xr0 = q == 0 ? 0.0 : sm[L - q].x;     // x_{M-2q}
    const double xr1 = sm[L - 1 - q].y;                // x_{M-2q-1}
    const double s0 = __ldg(&sinv[2 * q]), s1 = __ldg(&sinv[2 * q + 1]);
    v[m] = make_double2(fma(s0, a.x + xr0, 0.5 * (a.x - xr0)), fma(s1, a.y + xr1, 0.5 * (a.y - xr1)));
  }
}

// exclusive scan of a per-thread double over the sequence's T threads
template <int LOGL>
KFBI_DEV double scan_excl(const reg::View<LOGL> &sm, int t, double acc) {
  constexpr int T = reg::Cfg<LOGL>::T;
  static_assert(T >= 32 && T <= reg::Cfg<LOGL>::CTA_T, "one-CTA sequences");
  const int lane = threadIdx.x & 31;
  double inc = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  double off = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) off = 0.0;
  if constexpr (T > 32) {
    const int warp = t >> 5;
    if (lane == 31) sm.scr[0][warp] = make_double2(inc, 0.0);
    reg::seq_sync<LOGL>();
    double pw = 0.0;
    for (int w = 0; w < warp; ++w) pw += sm.scr[0][w].x;
    off += pw;
  }
  return off;
}

// Zc in sm (natural) -> out[c] = (C_2k, C_2k+1), k = 16 t + c
template <int LOGL>
KFBI_DEV void post(const reg::View<LOGL> &sm, int t, double2 (&out)[reg::E],
                   const double2 *__restrict__ twM) {
  constexpr int L = 1 << LOGL;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < reg::E; ++c) {
    const int k = reg::E * t + c;
    const double2 zk = sm[k];
    const double2 zm = sm[(L - k) & (L - 1)];
    const double ax = 0.5 * (zk.x + zm.x), ay = 0.5 * (zk.y - zm.y);
    const double bx = 0.5 * (zk.y + zm.y), by = -0.5 * (zk.x - zm.x);
    const double2 w = __ldg(&twM[k]);
    const double yx = ax + (w.x * bx - w.y * by);
    const double yy = ay + (w.x * by + w.y * bx);
    const double r = k == 0 ? yx : 2.0 * yx;
    acc = c == 0 ? r : acc + r;
    out[c] = make_double2(k == 0 ? 0.0 : -2.0 * yy, acc);
  }
  const double off = scan_excl<LOGL>(sm, t, acc);
#pragma unroll
  for (int c = 0; c < reg::E; ++c) out[c].y += off;
}

// staged pairs -> C pairs (out, natural pair index 16 t + c)
template <int LOGL>
KFBI_DEV void dst_staged(const reg::View<LOGL> &sm, int t, const BoxArgs &a, double2 (&out)[reg::E]) {
  double2 v[reg::E];
  pre<LOGL>(v, sm, t, a.sinv);
  reg::seq_sync<LOGL>();
  reg::fft<LOGL, 2>(v, sm, t, a.twg);          // length-L FFT from the length-M table
  post<LOGL>(sm, t, out, a.twg);
}

}  // namespace realdst

// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN - 1>::CTA_T, 1)
rows_fwd_real(BoxArgs a, const double *__restrict__ rhs, double sign, CorrArgs<double> corr) {
  constexpr int LOGL = LOGN - 1;
  using C = reg::Cfg<LOGL>;
  static_assert(C::S == 1 && C::CL == 1, "one sequence per CTA");
  constexpr int M = 1 << LOGN, L = C::N, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGL> sm = reg::make_view<LOGL>(smem, seq, t);
  const int stride = M + 1;
  const int r0 = blockIdx.x;                     // slab row
  const int j = a.row0 + r0;                     // grid row (0: zero ring)
  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) {
    const int q = t + m * TT;
    double x0 = 0.0, x1 = 0.0;
    if (j >= 1 && rhs != nullptr) {
      const double *row = rhs + (size_t)r0 * stride;
      if (q >= 1) x0 = row[2 * q];
      x1 = row[2 * q + 1];
    }
    v[m] = make_double2(x0 * sign, x1 * sign);
  }
  stage<LOGL>(sm, v, t);
  if (corr.jv && j >= 1) {
    reg::seq_sync<LOGL>();
    const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
    for (int g = g0 + t; g < g1; g += TT) {
      const double cv = group_correction<double>(corr, g);
      const int i = corr.group_node[g] - j * stride;
      reinterpret_cast<double *>(&sm[i >> 1])[i & 1] += cv;
    }
  }
  reg::seq_sync<LOGL>();
  double2 out[reg::E];
  realdst::dst_staged<LOGL>(sm, t, a, out);
  reg::seq_sync<LOGL>();
  unstage<LOGL>(sm, out, t);
  reg::seq_sync<LOGL>();
  // panel pp = slots 2pp, 2pp+1 of this row: 32 bytes
  for (int i = t; i < L; i += TT) *rows_fwd_dst(a, i >> 1, r0, i & 1) = sm[i];
}

// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN - 1>::CTA_T, 1) cols_real(BoxArgs a) {
  constexpr int LOGL = LOGN - 1;
  using C = reg::Cfg<LOGL>;
  constexpr int M = 1 << LOGN, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGL> sm = reg::make_view<LOGL>(smem, seq, t);
  const int q = blockIdx.x;                      // real column of this rank
  const int pl = q >> 2, w = q & 3;
  const int kx = 4 * (a.pp0 + pl) + w;           // spectral x index
  const int lr = 31 - __clz(a.rows);
  double *P = static_cast<double *>(a.panels);
  auto at = [&](int jj) -> double & {
    const size_t blk = (size_t)(jj >> lr) * a.npl + pl;
    return P[(blk * a.rows + (jj & (a.rows - 1))) * 4 + w];
  };
  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) {
    const int qq = t + m * TT;
    v[m] = make_double2(qq >= 1 ? at(2 * qq) : 0.0, at(2 * qq + 1));
  }
  stage<LOGL>(sm, v, t);
  reg::seq_sync<LOGL>();
  double2 out[reg::E];
  realdst::dst_staged<LOGL>(sm, t, a, out);
  // spectral division (boxsolve.py:74-76), p = 2k, 2k+1
  const double lq = a.lam[kx];
#pragma unroll
  for (int c = 0; c < reg::E; ++c) {
    const int p = 2 * (reg::E * t + c);
    const double x = p == 0 ? 0.0 : (out[c].x / ((a.lam[p] + lq) - a.kre)) * a.inv4m2;
    const double y = (out[c].y / ((a.lam[p + 1] + lq) - a.kre)) * a.inv4m2;
    out[c] = make_double2(x, y);
  }
  reg::seq_sync<LOGL>();
  unstage<LOGL>(sm, out, t);
  reg::seq_sync<LOGL>();
  realdst::dst_staged<LOGL>(sm, t, a, out);
  reg::seq_sync<LOGL>();
  unstage<LOGL>(sm, out, t);
  reg::seq_sync<LOGL>();
  // result element jj: in place, or into the row-pass buffer of its owner
  auto out_at = [&](int jj) -> double & {
    if (!a.dst[0]) return at(jj);
    return static_cast<double *>(a.dst[jj >> lr])[((size_t)(a.pp0 + pl) * a.rows + (jj & (a.rows - 1))) * 4 + w];
  };
  for (int qq = t; qq < M / 2; qq += TT) {
    const double2 s2 = sm[qq];
    out_at(2 * qq) = s2.x;
    out_at(2 * qq + 1) = s2.y;
  }
}

// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN - 1>::CTA_T, 1) rows_inv_real(BoxArgs a, double *__restrict__ u) {
  constexpr int LOGL = LOGN - 1;
  using C = reg::Cfg<LOGL>;
  constexpr int M = 1 << LOGN, L = C::N, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGL> sm = reg::make_view<LOGL>(smem, seq, t);
  const int stride = M + 1;
  const int r0 = blockIdx.x;
  const int j = a.row0 + r0;
  // FACR even rows nobody reads (trace-only / masked solves, per even row)
  if (a.row_step == 2 && a.row_need && !a.row_need[r0]) return;
  const double2 *P2 = static_cast<const double2 *>(a.panels);
  const size_t R = a.rows;
  for (int i = t; i < L; i += TT) {
    double2 s2 = P2[((size_t)(i >> 1) * R + r0) * 2 + (i & 1)];
    if (i == 0) s2.x = 0.0;                     // x_0 = 0
    sm[i] = s2;
  }
  reg::seq_sync<LOGL>();
  double2 out[reg::E];
  realdst::dst_staged<LOGL>(sm, t, a, out);
  reg::seq_sync<LOGL>();
  unstage<LOGL>(sm, out, t);
  reg::seq_sync<LOGL>();
  double *urow = u + (size_t)r0 * a.row_step * stride;   // row_step 2: FACR even rows
  for (int n = t; n <= M; n += TT) {
    double val = 0.0;
    if (j >= 1 && n >= 1 && n < M) {
      const double2 s2 = sm[n >> 1];
      val = (n & 1) ? s2.y : s2.x;
    }
    urow[n] = val;
    if (a.ring_end && r0 == a.rows - 1) urow[stride + n] = 0.0;
  }
}

}  // namespace kfbi
