// Box solve with the neumann-zero (mirror ghost) closure: DCT-I along x and
// y of the full (M+1)^2 rhs, divide by (lam_p + lam_q - kappa), p, q = 0..M,
// inverse DCT-I both ways (boxsolve.py:58-63, 66-94; rhs is read everywhere
// and the solution has no zero ring).  Same three-pass structure and
// register engine as the dirichlet-zero solve (box_reg.cuh) with the DCT-I
// pre/post-processing of dst_reg.cuh; M + 1 points per line, so the
// transform length N = M covers x_0..x_{M-1} in the sequence buffer and x_M
// in the extra slot.
//
// Panels: (M/4 + 1) real / (M/2 + 1) complex 32-byte strips of M + 1 rows,
// P2[(pp * (M+1) + j) * 2 + w]; row pairs (2q, 2q+1), q = 0..M/2 (the last
// pair has no second row).
#pragma once

#include "box_reg.cuh"

namespace kfbi {

// staged x_0..x_N -> C_0..C_N: out[c] = C_{16 t + c}, outN = C_N
template <int LOGN>
KFBI_DEV void dct_staged(const reg::View<LOGN> &sm, int t, const BoxArgs &a,
                         double2 (&out)[reg::E], double2 &outN) {
  constexpr int N = 1 << LOGN;
  double2 v[reg::E];
  const double2 c1 = reg::pre_dct<LOGN>(v, sm, t, a.sinv);
  reg::seq_sync<LOGN>();
  reg::fft<LOGN>(v, sm, t, a.twg);
  const double2 yh = sm[N / 2];
  outN = cadd(yh, yh);
  reg::post<LOGN, true>(sm, t, out, c1);
}

// out / outN back into the sequence buffer (natural order)
template <int LOGN>
KFBI_DEV void unstage_n(const reg::View<LOGN> &sm, const double2 (&out)[reg::E], double2 outN, int t) {
  unstage<LOGN>(sm, out, t);
  if (t == 0) *sm.ext = outN;
}

template <int LOGN>
KFBI_DEV double2 slot_n(const reg::View<LOGN> &sm, int n) {
  constexpr int N = 1 << LOGN;
  return n < N ? sm[n] : (n == N ? *sm.ext : make_double2(0.0, 0.0));
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB)
rows_fwd_neu(BoxArgs a, const void *__restrict__ rhs, double sign,
             CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  constexpr int RR = M + 1;                       // panel rows
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int stride = M + 1;
  const int q = seq_index<LOGN>(seq);
  const int nseq = CPLX ? M + 1 : M / 2 + 1;
  const bool valid = q < nseq;
  const int j0 = CPLX ? q : 2 * q;
  const bool has2 = !CPLX && j0 + 1 <= M;

  auto load = [&](int n) -> double2 {
    double2 w = make_double2(0.0, 0.0);
    if (valid && rhs != nullptr) {
      if (CPLX) {
        w = static_cast<const double2 *>(rhs)[(size_t)j0 * stride + n];
      } else {
        const double *r = static_cast<const double *>(rhs);
        w.x = r[(size_t)j0 * stride + n];
        if (has2) w.y = r[(size_t)(j0 + 1) * stride + n];
      }
    }
    return cscale(w, sign);
  };
  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) v[m] = load(t + m * TT);
  stage<LOGN>(sm, v, t);
  if (t == 0) *sm.ext = load(M);
  if (corr.jv) {
    reg::seq_sync<LOGN>();
    if (valid) {
      const int nrows = has2 ? 2 : 1;
      for (int qq = 0; qq < nrows; ++qq) {
        const int j = j0 + qq;
        const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
        for (int g = g0 + t; g < g1; g += TT) {
          const T cv = group_correction<T>(corr, g);
          const int i = corr.group_node[g] - j * stride;
          double2 &slot = i < M ? sm[i] : *sm.ext;
          if constexpr (CPLX) slot = cadd(slot, cv);
          else reinterpret_cast<double *>(&slot)[qq] += cv;
        }
      }
    }
  }
  reg::seq_sync<LOGN>();
  double2 out[reg::E], outN;
  dct_staged<LOGN>(sm, t, a, out, outN);
  reg::seq_sync<LOGN>();
  unstage_n<LOGN>(sm, out, outN, t);
  reg::seq_sync<LOGN>();
  if (valid) {
    double2 *P2 = static_cast<double2 *>(a.panels);
    if (!CPLX) {
      for (int i = t; i < 4 * (M / 4 + 1); i += TT) {
        const int pp = i >> 2, part = i & 3, row = part >> 1;
        if (row && !has2) continue;
        const int n0 = 4 * pp + 2 * (part & 1);
        const double2 v0 = slot_n<LOGN>(sm, n0), v1 = slot_n<LOGN>(sm, n0 + 1);
        P2[((size_t)pp * RR + j0 + row) * 2 + (part & 1)] =
            row ? make_double2(v0.y, v1.y) : make_double2(v0.x, v1.x);
      }
    } else {
      for (int i = t; i < 2 * (M / 2 + 1); i += TT)
        P2[((size_t)(i >> 1) * RR + j0) * 2 + (i & 1)] = slot_n<LOGN>(sm, i);
    }
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB) cols_neu(BoxArgs a) {
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  constexpr int RR = M + 1;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int q = seq_index<LOGN>(seq);
  const int np = CPLX ? M / 2 + 1 : M / 4 + 1;
  const bool valid = q < 2 * np;
  const int pp = q >> 1, half = q & 1;
  double2 *col = static_cast<double2 *>(a.panels) + (size_t)pp * RR * 2 + half;

  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) {
    const int n = t + m * TT;
    v[m] = valid ? col[2 * n] : make_double2(0.0, 0.0);
  }
  stage<LOGN>(sm, v, t);
  if (t == 0) *sm.ext = valid ? col[2 * M] : make_double2(0.0, 0.0);
  reg::seq_sync<LOGN>();
  double2 out[reg::E], outN;
  dct_staged<LOGN>(sm, t, a, out, outN);

  // spectral division, p, kx = 0..M (boxsolve.py:38-44, 74-76)
  auto scale = [&](double2 w, int p) -> double2 {
    const double lp = a.lam[p];
    if (!CPLX) {
      const int kx = 4 * pp + 2 * half;
      const double x = kx <= M ? (w.x / ((lp + a.lam[kx]) - a.kre)) * a.inv4m2 : 0.0;
      const double y = kx + 1 <= M ? (w.y / ((lp + a.lam[kx + 1]) - a.kre)) * a.inv4m2 : 0.0;
      return make_double2(x, y);
    } else {
      const int kx = 2 * pp + half;
      if (kx > M) return make_double2(0.0, 0.0);
      return cscale(cdiv(w, make_double2((lp + a.lam[kx]) - a.kre, -a.kim)), a.inv4m2);
    }
  };
#pragma unroll
  for (int c = 0; c < reg::E; ++c) out[c] = scale(out[c], reg::E * t + c);
  outN = scale(outN, M);
  reg::seq_sync<LOGN>();
  unstage_n<LOGN>(sm, out, outN, t);
  reg::seq_sync<LOGN>();
  dct_staged<LOGN>(sm, t, a, out, outN);
  reg::seq_sync<LOGN>();
  unstage_n<LOGN>(sm, out, outN, t);
  reg::seq_sync<LOGN>();
  if (valid)
    for (int n = t; n <= M; n += TT) col[2 * n] = slot_n<LOGN>(sm, n);
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB)
rows_inv_neu(BoxArgs a, void *__restrict__ u) {
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  constexpr int RR = M + 1;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int stride = M + 1;
  const int q = seq_index<LOGN>(seq);
  const int nseq = CPLX ? M + 1 : M / 2 + 1;
  const bool valid = q < nseq;
  const int j0 = CPLX ? q : 2 * q;
  const bool has2 = !CPLX && j0 + 1 <= M;
  const double2 *P2 = static_cast<const double2 *>(a.panels);

  auto load = [&](int n) -> double2 {
    if (!valid) return make_double2(0.0, 0.0);
    if (CPLX) return P2[((size_t)(n >> 1) * RR + j0) * 2 + (n & 1)];
    const double *s0 = reinterpret_cast<const double *>(P2) + ((size_t)(n >> 2) * RR + j0) * 4 + (n & 3);
    return make_double2(s0[0], has2 ? s0[4] : 0.0);
  };
  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) v[m] = load(t + m * TT);
  stage<LOGN>(sm, v, t);
  if (t == 0) *sm.ext = load(M);
  reg::seq_sync<LOGN>();
  double2 out[reg::E], outN;
  dct_staged<LOGN>(sm, t, a, out, outN);
  reg::seq_sync<LOGN>();
  unstage_n<LOGN>(sm, out, outN, t);
  reg::seq_sync<LOGN>();
  if (valid) {
    if (!CPLX) {
      double *U = static_cast<double *>(u);
      double *u0 = U + (size_t)j0 * stride;
      for (int n = t; n <= M; n += TT) {
        const double2 w = slot_n<LOGN>(sm, n);
        u0[n] = w.x;
        if (has2) u0[stride + n] = w.y;
      }
    } else {
      double2 *U = static_cast<double2 *>(u);
      for (int n = t; n <= M; n += TT) U[(size_t)j0 * stride + n] = slot_n<LOGN>(sm, n);
    }
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

}  // namespace kfbi
