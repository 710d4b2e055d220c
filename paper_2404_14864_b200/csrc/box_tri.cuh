// Column pass of the dirichlet-zero box solve as constant-coefficient
// tridiagonal solves along y (the "FA + tridiagonal" form of the fast
// Helmholtz solver) instead of DST-I -> divide -> DST-I.
//
// The reference's column stage (boxsolve.py:70-82, scipy dst / idst along
// axis 0 between the row transforms) computes, for every spectral x index kx,
//
//   out = DST_y( DST_y(P) / (lam_kx + lam_q - kappa) ) / (4 M^2)
//       = Tri_kx^{-1} P / (2 M),
//
// because DST-I diagonalises the 1-D three-point Laplacian with a zero ring:
// Tri_kx y_j = (y_{j-1} - 2 y_j + y_{j+1}) / h^2 + (lam_kx - kappa) y_j,
// j = 1..M-1, y_0 = y_M = 0 (lam_q are exactly its eigenvalues).  The same
// linear map is applied here by a factored recurrence, O(M) per column
// instead of two length-M FFTs, so the pass is HBM-bound:
//
//   r: the root of r^2 + b r + 1 = 0 with |r| < 1, b = -2 + (lam_kx - kappa) h^2
//   y_{j-1} + b y_j + y_{j+1} = -(1/r)(1 - rE)(1 - rE^{-1}) y
//   forward  v_j = r v_{j-1} - P_j          (v_0 = 0)
//   backward z_j = r z_{j+1} + v_j          (z_M = 0)
//   out_j = A z_j + B (r^j - r^{2M-j}),  A = r h^2 / (2M),
//           B = -A r z_1 / (1 - r^{2M})     (restores y_0 = 0 exactly)
//
// Both recurrences contract (|r| < 1), so rounding does not grow; against a
// long-double solve of the same system this is more accurate than the FFT
// route (2e-14 vs 7e-13 relative at M = 1024, kappa = 3.7).
//
// Parallel form: a thread owns CH consecutive rows of one 16-byte column
// slot (two real columns, or one complex column) in registers; each
// recurrence is a local sweep from zero, an affine scan of the chunk carries
// (multiplier r^CH: warp shuffles, then the warp totals through shared
// memory), and a fix-up with the running powers of r.  HBM traffic: the
// panel strip is read once and written once (2 (M-1)^2 s bytes per launch).
// Same panel layout and slab / peer-store conventions as cols_reg.
#pragma once

#include "box_kernels.cuh"

namespace kfbi {
namespace tri {

// a * b and a * b + c on the 16-byte slot: two independent real columns
// (componentwise) or one complex column.
template <bool CPLX>
KFBI_DEV double2 mul(double2 a, double2 b) {
  if constexpr (CPLX) return cmul(a, b);
  else return make_double2(a.x * b.x, a.y * b.y);
}
template <bool CPLX>
KFBI_DEV double2 mad(double2 a, double2 b, double2 c) {
  if constexpr (CPLX)
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
  else return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
template <bool CPLX>
KFBI_DEV double2 one() {
  return CPLX ? make_double2(1.0, 0.0) : make_double2(1.0, 1.0);
}
// a^e, e >= 0, by binary powering (e <= 2^15)
template <bool CPLX>
KFBI_DEV double2 pw(double2 a, int e) {
  double2 acc = one<CPLX>();
  while (e) {
    if (e & 1) acc = mul<CPLX>(acc, a);
    a = mul<CPLX>(a, a);
    e >>= 1;
  }
  return acc;
}

KFBI_DEV double2 csqrt_(double2 z) {
  const double m = hypot(z.x, z.y);
  if (m == 0.0) return make_double2(0.0, 0.0);
  const double t = sqrt(0.5 * (m + fabs(z.x)));
  if (z.x >= 0.0) return make_double2(t, z.y / (2.0 * t));
  return make_double2(fabs(z.y) / (2.0 * t), copysign(t, z.y));
}

// Root with |r| < 1 of r^2 + b r + 1 = 0, b = -2 - 2 bm1:
// r = 1 / (beta + sqrt(beta^2 - 1)), beta = 1 + bm1, beta^2 - 1 = bm1 (beta + 1)
// (formed without cancellation; the branch with |beta + s| >= |beta - s|).
KFBI_DEV double root_real(double bm1) {
  const double beta = 1.0 + bm1;
  return 1.0 / (beta + sqrt(bm1 * (beta + 1.0)));
}
KFBI_DEV double2 root_cplx(double2 bm1) {
  const double2 beta = make_double2(1.0 + bm1.x, bm1.y);
  double2 s = csqrt_(cmul(bm1, make_double2(beta.x + 1.0, beta.y)));
  if (beta.x * s.x + beta.y * s.y < 0.0) s = cneg(s);
  return cdiv(make_double2(1.0, 0.0), cadd(beta, s));
}

template <int LOGM>
struct Cfg {
  static constexpr int M = 1 << LOGM;
#ifndef KFBI_TRI_CH
  static constexpr int CH = M >= 512 ? 32 : M / 16;      // rows per thread
#else
  static constexpr int CH = M >= 512 ? KFBI_TRI_CH : M / 16;
#endif
#ifndef KFBI_TRI_NH1_FROM
  static constexpr int NH = M >= 8192 ? 1 : 2;          // 16-byte slots per CTA
#else
  static constexpr int NH = M >= KFBI_TRI_NH1_FROM ? 1 : 2;
#endif
  static constexpr int NCH = M / CH;                    // chunks per column
  static constexpr int THREADS = NCH * NH;
  static constexpr int CPW = 32 / NH;                   // chunks of one slot per warp
  static constexpr int NW = NCH / CPW;                  // warps per slot
  static constexpr int LCPW = NH == 1 ? 5 : 4;
#ifndef KFBI_TRI_REGS
  static constexpr int REGS = 168;                      // register budget per thread
#else
  static constexpr int REGS = KFBI_TRI_REGS;
#endif
  static constexpr int MINB0 = 65536 / (THREADS * REGS);
  static constexpr int MINB = MINB0 < 1 ? 1 : MINB0;    // CTAs per SM
  static_assert(THREADS >= 32 && THREADS <= 1024, "tri column pass: CTA size");
  static_assert(NCH % CPW == 0, "whole warps per slot");
};

}  // namespace tri

// Shared memory of the scans of one CTA (NH slots, NW warps per slot).
constexpr int TRI_NPOW = 12;                     // r^(CH 2^s), s < 12 (exponents < 2^12 CH)
template <int NH, int NW>
struct TriSmem {
  double2 tot[NH][NW];
  double2 z1s[NH];
  double2 rcs[NH][TRI_NPOW];
  double2 w0s[NH];
};

// The recurrences of one thread's CH rows [j0, j0 + CH) of column slot
// (pp, half) held in x (in place).  Every thread of the CTA calls it (CTA
// barriers inside).  With local sweeps from zero
//   vL_i = r vL_{i-1} - P_i,   zL_i = r zL_{i+1} + vL_i
// the exact chunk values are v_i = vL_i + r^{i+1} V and
// z_i = zL_i + V w_i + Z r^{CH-i}, w_i = sum_{m>=i} r^{2m-i+1}
// = (r^{i+1} - r^{2CH-i+1}) / (1 - r^2), where V (true v at row j0 - 1) and
// Z (true z at row j0 + CH) come from two affine scans over the chunks: the
// forward one of the local ends vL_{CH-1}, the backward one of the chunk
// starts zL_0 + V w_0.  Both local sweeps run back to back; the epilogue
//   out_i = A z_i + B (r^j - r^{2M-j}) = A zL_i + alpha r^i + gamma r^{CH-1-i}
// is two multiply chains.
// Row slabs across ranks (cols_tri_dist): the rank's R = 2^LOGM rows are
// solved with zero carries at the slab ends, the three slab aggregates of
// every column (v at the last row, z at the first row, z at global row 1)
// are pushed to every rank over peer memory, and each rank folds the other
// slabs' carries into its epilogue.  nullptr: one slab holds all rows.
struct TriDist {
  int P, g;                                   // ranks, this rank
  int units;                                  // column units (strips or half strips)
  int virt;                                   // 1: all ranks in one launch (blockIdx.y = rank)
  unsigned long long epoch;
  long long max_spins;
  int *timed_out;
  void *vpanels[8];                           // virt: every rank's panel buffer
  double2 *agg[8];                            // [unit][P][NH][3] of rank h, as mapped here
  unsigned long long *flg[8];                 // [unit][P] of rank h, as mapped here
};

template <bool CPLX, class C, bool DIST = false>
KFBI_DEV void tri_solve_c(double2 (&x)[C::CH], const BoxArgs &a, int pp, int half, int hs, int chunk,
                          TriSmem<C::NH, C::NW> &sh, const TriDist *dd = nullptr, int unit = 0,
                          int g = 0) {
  constexpr int CH = C::CH, NH = C::NH, CPW = C::CPW, NW = C::NW, NCH = C::NCH;
  static_assert(2 * NCH < (1 << TRI_NPOW), "power table");
  const int cw = chunk & (CPW - 1);              // chunk index within the warp
  const int wv = chunk / CPW;                    // warp index within the slot
  // per-column root r (a.trow: one root for the x recurrence of a grid row;
  // a.red: the even-row system's root r^2)
  const double hh2 = 0.5 * a.h2;
  double2 r;
  int kx0;
  if (a.trow) {
    kx0 = 1;
    if constexpr (CPLX) r = tri::root_cplx(make_double2(a.tb_re, a.tb_im));
    else {
      const double rr = tri::root_real(a.tb_re);
      r = make_double2(rr, rr);
    }
  } else if constexpr (CPLX) {
    kx0 = 2 * pp + half;
    r = tri::root_cplx(make_double2((a.kre - a.lam[kx0]) * hh2, a.kim * hh2));
    if (kx0 == 0) r = make_double2(0.0, 0.0);
  } else {
    kx0 = 4 * pp + 2 * half;
    r = make_double2(kx0 == 0 ? 0.0 : tri::root_real((a.kre - a.lam[kx0]) * hh2),
                     tri::root_real((a.kre - a.lam[kx0 + 1]) * hh2));
  }
  if (a.red) r = tri::mul<CPLX>(r, r);
  const double2 zero = make_double2(0.0, 0.0);

  // ---- local sweeps (no dependence on other chunks) ------------------------
  double2 e = zero;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    e = tri::mad<CPLX>(r, e, cneg(x[i]));
    x[i] = e;                                    // vL
  }
  const double2 eF = e;                          // vL_{CH-1}
  e = zero;
#pragma unroll
  for (int i = CH - 1; i >= 0; --i) {
    e = tri::mad<CPLX>(r, e, x[i]);
    x[i] = e;                                    // zL
  }
  const double2 sL = e;                          // zL_0

  // per-slot powers r^(CH 2^s) and w_0 = sum_{m<CH} r^{2m+1} (chunk 0, shared)
  if (chunk == 0) {
    double2 q = tri::pw<CPLX>(r, CH);
#pragma unroll
    for (int s2 = 0; s2 < TRI_NPOW; ++s2) {
      sh.rcs[hs][s2] = q;
      q = tri::mul<CPLX>(q, q);
    }
    const double2 r2 = tri::mul<CPLX>(r, r);
    double2 w = zero;
#pragma unroll 4
    for (int m = CH - 1; m >= 0; --m) w = tri::mad<CPLX>(r2, w, r);   // Horner: r sum r^{2m}
    sh.w0s[hs] = w;
  }
  __syncthreads();
  auto rc2 = [&](int s2) -> double2 { return sh.rcs[hs][s2]; };
  auto rc_pow = [&](int ex) -> double2 {        // r^(CH ex), 0 <= ex < 2^TRI_NPOW
    double2 acc = tri::one<CPLX>();
#pragma unroll
    for (int s2 = 0; s2 < TRI_NPOW; ++s2)
      if (ex & (1 << s2)) acc = tri::mul<CPLX>(acc, rc2(s2));
    return acc;
  };
  const int sl = NH;                             // lane stride between chunks of a slot

  // ---- forward carries: I_k = eF_k + r^CH I_{k-1}, V_k = I_{k-1} ----------
  double2 I = eF;
#pragma unroll
  for (int s2 = 0; s2 < C::LCPW; ++s2) {
    const int d = 1 << s2;
    double2 y;
    y.x = __shfl_up_sync(0xffffffffu, I.x, d * sl);
    y.y = __shfl_up_sync(0xffffffffu, I.y, d * sl);
    if (cw >= d) I = tri::mad<CPLX>(rc2(s2), y, I);
  }
  double2 V;
  {
    double2 acc = zero;                          // carry into this warp
    if constexpr (NW > 1) {
      if (cw == CPW - 1) sh.tot[hs][wv] = I;
      __syncthreads();
      const double2 rw = rc_pow(CPW);
      for (int w = 0; w < wv; ++w) acc = tri::mad<CPLX>(rw, acc, sh.tot[hs][w]);
      I = tri::mad<CPLX>(rc_pow(cw + 1), acc, I);
    }
    V.x = __shfl_up_sync(0xffffffffu, I.x, sl);
    V.y = __shfl_up_sync(0xffffffffu, I.y, sl);
    if (cw == 0) V = acc;
  }

  // ---- backward carries: J_k = s_k + r^CH J_{k+1}, s_k = zL_0 + V w_0 -----
  double2 J = tri::mad<CPLX>(V, sh.w0s[hs], sL);
#pragma unroll
  for (int s2 = 0; s2 < C::LCPW; ++s2) {
    const int d = 1 << s2;
    double2 y;
    y.x = __shfl_down_sync(0xffffffffu, J.x, d * sl);
    y.y = __shfl_down_sync(0xffffffffu, J.y, d * sl);
    if (cw + d < CPW) J = tri::mad<CPLX>(rc2(s2), y, J);
  }
  double2 Z;                                     // true z at row j0 + CH
  {
    double2 acc = zero;                          // carry into this warp from below
    if constexpr (NW > 1) {
      __syncthreads();                           // forward totals consumed
      if (cw == 0) sh.tot[hs][wv] = J;
      __syncthreads();
      const double2 rw = rc_pow(CPW);
      for (int w = NW - 1; w > wv; --w) acc = tri::mad<CPLX>(rw, acc, sh.tot[hs][w]);
      J = tri::mad<CPLX>(rc_pow(CPW - cw), acc, J);
    }
    Z.x = __shfl_down_sync(0xffffffffu, J.x, sl);
    Z.y = __shfl_down_sync(0xffffffffu, J.y, sl);
    if (cw == CPW - 1) Z = acc;
  }

  // ---- slab carries (DIST) and the boundary term ---------------------------
  // z_i = zL_i + Vc w_i + Zc r^{CH-i} + Vg W_i + Zg r^{R-iota}, iota = chunk CH + i
  // (w, W: the chunk / slab sums r^{2m-i+1}); single slab: Vg = Zg = 0.
  const double2 rch = rc2(0);                    // r^CH
  const int P = DIST ? dd->P : 1;
  const int NT = P * NCH;                        // chunks of the whole column (M / CH)
  double2 Vg = zero, Zg = zero, z1;
  double2 inv1mr2;                               // 1 / ((1 - r)(1 + r))
  {
    const double2 d = tri::mul<CPLX>(make_double2(1.0 - r.x, -r.y),
                                     CPLX ? make_double2(1.0 + r.x, r.y) : make_double2(1.0 + r.y, 0.0));
    if constexpr (CPLX) inv1mr2 = cdiv(make_double2(1.0, 0.0), d);
    else inv1mr2 = make_double2(1.0 / ((1.0 - r.x) * (1.0 + r.x)), 1.0 / ((1.0 - r.y) * (1.0 + r.y)));
  }
  // rank-local z at row 1 of this slab's chunk 0 (global row 1 on rank 0)
  if (CH > 1 && chunk == 0) sh.z1s[hs] = tri::mad<CPLX>(Z, tri::pw<CPLX>(r, CH - 1), x[CH > 1 ? 1 : 0]);
  if (CH == 1 && chunk == 1) sh.z1s[hs] = tri::mad<CPLX>(V, sh.w0s[hs], tri::mad<CPLX>(Z, r, x[0]));
  if constexpr (DIST) {
    // slab aggregates: v at the last row (inclusive forward carry of the last
    // chunk), z at the first row (backward carry of chunk 0), z at row 1
    __shared__ double2 aggs[2][2];
    if (chunk == NCH - 1) aggs[hs][0] = I;
    if (chunk == 0) aggs[hs][1] = J;
    __syncthreads();
    if (threadIdx.x < NH) {                      // one thread per half: push to every rank
      const int h2 = threadIdx.x;
      const double2 v3[3] = {aggs[h2][0], aggs[h2][1], sh.z1s[h2]};
      for (int q = 0; q < P; ++q) {
        double2 *dst = dd->agg[q] + (((size_t)unit * P + g) * NH + h2) * 3;
        for (int k3 = 0; k3 < 3; ++k3) dst[k3] = v3[k3];
      }
      __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int q = 0; q < P; ++q) {
        unsigned long long *f = dd->flg[q] + (size_t)unit * P + g;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(dd->epoch) : "memory");
      }
      const unsigned long long *mine = dd->flg[g] + (size_t)unit * P;
      for (int q = 0; q < P; ++q) {
        for (long long it = 0;; ++it) {
          unsigned long long v;
          asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + q) : "memory");
          if (v >= dd->epoch) break;
          if (it >= dd->max_spins) {
            if (dd->timed_out) atomicExch(dd->timed_out, 1);
            break;
          }
          __nanosleep(32);
        }
      }
      __threadfence();
    }
    __syncthreads();
    // carries across slabs from the P aggregates of this column (own buffer)
    const double2 *ag = dd->agg[g] + (size_t)unit * P * NH * 3;
    const double2 rR = rc_pow(NCH);              // r^R
    // W_0 = (r - r^{2R+1}) / (1 - r^2)
    const double2 W0 = tri::mul<CPLX>(tri::mad<CPLX>(cneg(rc_pow(2 * NCH)), r, r), inv1mr2);
    double2 Vq = zero;                           // forward carry into slab q
    double2 sq[8];
    for (int q = 0; q < P; ++q) {
      const double2 eq = __ldcg(&ag[((size_t)q * NH + hs) * 3 + 0]);
      const double2 sLq = __ldcg(&ag[((size_t)q * NH + hs) * 3 + 1]);
      if (q == g) Vg = Vq;
      sq[q] = tri::mad<CPLX>(Vq, W0, sLq);      // z at slab q's first row without Z_q
      Vq = tri::mad<CPLX>(rR, Vq, eq);
    }
    double2 Zq = zero;                           // backward carry into slab q from below
    double2 Z0 = zero;
    for (int q = P - 1; q >= 0; --q) {
      if (q == g) Zg = Zq;
      if (q == 0) Z0 = Zq;
      Zq = tri::mad<CPLX>(rR, Zq, sq[q]);
    }
    // z_1 = zl1(slab 0) + Z_0 r^{R-1}
    z1 = tri::mad<CPLX>(Z0, tri::mul<CPLX>(rc_pow(NCH - 1), tri::pw<CPLX>(r, CH - 1)),
                        __ldcg(&ag[(size_t)hs * 3 + 2]));
  } else {
    __syncthreads();
    z1 = sh.z1s[hs];
  }
  const double sc = a.trow ? a.tscale : a.h2 / (2.0 * a.m);
  const double2 A = tri::mul<CPLX>(r, CPLX ? make_double2(sc, 0.0) : make_double2(sc, sc));
  const double2 r2m = rc_pow(2 * NT);            // r^{2M}
  double2 B;                                     // -A r z1 / (1 - r^2M)
  {
    const double2 num = tri::mul<CPLX>(tri::mul<CPLX>(A, r), z1);
    if constexpr (CPLX) {
      B = cneg(cdiv(num, make_double2(1.0 - r2m.x, -r2m.y)));
    } else {
      B = make_double2(-num.x / (1.0 - r2m.x), -num.y / (1.0 - r2m.y));
      if (kx0 == 0) B.x = 0.0;
    }
  }
  // alpha = A (Vc r + Vg r^{iota0+1}) / (1 - r^2) + B r^{j0}
  // gamma = A [-(Vc r^{CH+2} + Vg r^{2R-iota0-CH+2}) / (1 - r^2) + Zc r + Zg r^{R-iota0-CH+1}]
  //         - B r^{2M-j0-CH+1},   iota0 = chunk CH, j0 = g R + iota0
  const int gch = g * NCH + chunk;               // global chunk index
  const double2 Aq = tri::mul<CPLX>(A, inv1mr2);
  double2 Vsum = tri::mad<CPLX>(Vg, tri::mul<CPLX>(rc_pow(chunk), r), tri::mul<CPLX>(V, r));
  const double2 alpha = tri::mad<CPLX>(Aq, Vsum, tri::mul<CPLX>(B, rc_pow(gch)));
  const double2 r2 = tri::mul<CPLX>(r, r);
  double2 Vg2 = tri::mad<CPLX>(Vg, tri::mul<CPLX>(rc_pow(2 * NCH - chunk - 1), r2),
                               tri::mul<CPLX>(V, tri::mul<CPLX>(tri::mul<CPLX>(rch, r), r)));
  double2 gamma = tri::mul<CPLX>(Aq, Vg2);
  gamma = tri::mad<CPLX>(tri::mul<CPLX>(A, tri::mad<CPLX>(Zg, tri::mul<CPLX>(rc_pow(NCH - chunk - 1), r),
                                                          tri::mul<CPLX>(Z, r))),
                         tri::one<CPLX>(), cneg(gamma));
  gamma = tri::mad<CPLX>(cneg(B), tri::mul<CPLX>(rc_pow(2 * NT - gch - 1), r), gamma);
  {
    double2 c = alpha;                           // alpha r^i
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      x[i] = tri::mad<CPLX>(A, x[i], c);
      c = tri::mul<CPLX>(c, r);
    }
    c = gamma;                                   // gamma r^{CH-1-i}
#pragma unroll
    for (int i = CH - 1; i >= 0; --i) {
      x[i] = cadd(x[i], c);
      c = tri::mul<CPLX>(c, r);
    }
  }
  if (kx0 == 0) {                                // padding column kx = 0
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if constexpr (CPLX) x[i] = zero;
      else x[i].x = 0.0;
    }
  }
}

template <bool CPLX, int LOGM, bool DIST = false>
KFBI_DEV void tri_solve(double2 (&x)[tri::Cfg<LOGM>::CH], const BoxArgs &a, int pp, int half, int hs,
                        int chunk, TriSmem<tri::Cfg<LOGM>::NH, tri::Cfg<LOGM>::NW> &sh,
                        const TriDist *dd = nullptr, int unit = 0, int g = 0) {
  tri_solve_c<CPLX, tri::Cfg<LOGM>, DIST>(x, a, pp, half, hs, chunk, sh, dd, unit, g);
}

template <bool CPLX, int LOGM>
__global__ void __launch_bounds__(tri::Cfg<LOGM>::THREADS, tri::Cfg<LOGM>::MINB) cols_tri(BoxArgs a) {
  using C = tri::Cfg<LOGM>;
  constexpr int CH = C::CH, NH = C::NH;
  __shared__ TriSmem<NH, C::NW> sh;
  if (a.done && *a.done) return;
  const int t = threadIdx.x;
  const int half = NH == 2 ? (t & 1) : (blockIdx.x & 1);
  const int hs = NH == 2 ? half : 0;            // slot index in shared memory
  const int chunk = NH == 2 ? (t >> 1) : t;
  const int pl = NH == 2 ? blockIdx.x : (blockIdx.x >> 1);
  if (pl >= a.npl) return;                       // whole CTA: uniform
  const int pp = a.pp0 + pl;
  // rows [j0, j0 + CH) of the slot: one rank block (CH divides the slab rows),
  // 32 bytes apart
  const int j0 = chunk * CH;
  const int lr = 31 - __clz(a.rows);
  const int jb = j0 & (a.rows - 1);
  const double2 *src = static_cast<const double2 *>(a.panels) +
                       ((((size_t)(j0 >> lr) * a.npl + pl) * a.rows + jb) * 2 + half);
  double2 *dst = a.dst[0] ? static_cast<double2 *>(a.dst[j0 >> lr]) + (((size_t)pp * a.rows + jb) * 2 + half)
                          : const_cast<double2 *>(src);
  double2 x[CH];
  // FACR: rows flagged zero by the forward pass are not loaded (their panels
  // were not written)
  const unsigned char *rz = a.rowz;
#pragma unroll
  for (int i = 0; i < CH; ++i)
    x[i] = (j0 + i >= 1 && !(rz && rz[j0 + i])) ? src[2 * i] : make_double2(0.0, 0.0);
  tri_solve<CPLX, LOGM>(x, a, pp, half, hs, chunk, sh);
#pragma unroll
  for (int i = 0; i < CH; ++i) dst[2 * i] = (j0 + i >= 1) ? x[i] : make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// Column stage of the slab-decomposed box solve WITHOUT transposes: rank g
// keeps its R = 2^LOGR rows of every spectral column (the row pass's own
// panel layout [pp][R][w]), solves them with zero carries at the slab ends
// and exchanges three values per column with the other ranks over peer
// memory inside the kernel (TriDist).  Persistent CTAs walk the column units
// in the same order on every rank, so the partner CTAs of a unit are always
// resident (cooperative launch) and the per-unit flag waits cannot deadlock.
// Traffic between GPUs: 3 P values per column instead of two all-to-alls of
// M^2 s / P bytes per rank.
template <bool CPLX, int LOGR>
__global__ void __launch_bounds__(tri::Cfg<LOGR>::THREADS, 1) cols_tri_dist(BoxArgs a, TriDist d) {
  using C = tri::Cfg<LOGR>;
  constexpr int CH = C::CH, NH = C::NH, R = C::M;
  __shared__ TriSmem<NH, C::NW> sh;
  if (a.done && *a.done) return;
  const int t = threadIdx.x;
  const int g = d.virt ? (int)blockIdx.y : d.g;
  const int chunk = NH == 2 ? (t >> 1) : t;
  const int j0 = chunk * CH;
  double2 *panels = static_cast<double2 *>(d.virt ? d.vpanels[g] : a.panels);
  for (int unit = blockIdx.x; unit < d.units; unit += gridDim.x) {
    const int half = NH == 2 ? (t & 1) : (unit & 1);
    const int pl = NH == 2 ? unit : (unit >> 1);
    double2 *col = panels + (((size_t)pl * R + j0) * 2 + half);
    double2 x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = (g == 0 && j0 + i == 0) ? make_double2(0.0, 0.0) : col[2 * i];
    tri_solve<CPLX, LOGR, true>(x, a, pl, half, NH == 2 ? half : 0, chunk, sh, &d, unit, g);
#pragma unroll
    for (int i = 0; i < CH; ++i) col[2 * i] = (g == 0 && j0 + i == 0) ? make_double2(0.0, 0.0) : x[i];
    __syncthreads();                             // shared scan state reused by the next unit
  }
}

// ---------------------------------------------------------------------------
// M = 4096: one persistent CTA per SM walks the strips; while it solves strip
// s from registers, the bulk-copy engine (cp.async.bulk, mbarrier completion)
// already streams strip s + grid into shared memory, so HBM reads overlap the
// recurrences and the stores.  The strip (M rows x 32 bytes, contiguous) is
// copied as 1 KB chunks (the 32 rows of one thread pair) to 1056-byte slots:
// the 16-byte reads of a quarter warp then hit 8 distinct bank groups.
namespace tri {
constexpr int TMA_LOGM = 12;
constexpr int TMA_SLOT = 1056;                      // bytes per 32-row chunk in smem
constexpr int TMA_SMEM = (1 << TMA_LOGM) / 32 * TMA_SLOT;

KFBI_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
KFBI_DEV void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
KFBI_DEV void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
KFBI_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
KFBI_DEV void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace tri

template <bool CPLX>
__global__ void __launch_bounds__(tri::Cfg<tri::TMA_LOGM>::THREADS, 1) cols_tri_tma(BoxArgs a) {
  constexpr int LOGM = tri::TMA_LOGM;
  using C = tri::Cfg<LOGM>;
  constexpr int CH = C::CH, NH = C::NH, NCH = C::NCH;
  static_assert(NH == 2 && CH == 32, "bulk-copy column pass: thread pairs own 32-row chunks");
  extern __shared__ __align__(128) unsigned char tbuf[];
  __shared__ TriSmem<NH, C::NW> sh;
  __shared__ __align__(8) uint64_t bar;
  if (a.done && *a.done) return;
  const int t = threadIdx.x;
  const int half = t & 1, chunk = t >> 1;
  const int lr = 31 - __clz(a.rows);
  auto chunk_src = [&](int pl, int k) -> const unsigned char * {
    const int j = k * CH;
    const size_t blk = (size_t)(j >> lr) * a.npl + pl;
    return reinterpret_cast<const unsigned char *>(a.panels) + ((blk * a.rows + (j & (a.rows - 1))) * 32);
  };
  auto issue = [&](int pl) {                     // warp 0: 128 chunk copies of 1 KB
    if (t < 32) {
      if (t == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tri::mbar_arrive_tx(&bar, NCH * 1024);
      }
      __syncwarp();
      for (int k = t; k < NCH; k += 32) tri::bulk_g2s(tbuf + k * tri::TMA_SLOT, chunk_src(pl, k), 1024, &bar);
    }
  };
  if (t == 0) {
    tri::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;
  int pl = blockIdx.x;
  if (pl < a.npl) issue(pl);
  for (; pl < a.npl; pl += gridDim.x) {
    tri::mbar_wait(&bar, parity);
    parity ^= 1;
    double2 x[CH];
    const unsigned char *mine = tbuf + chunk * tri::TMA_SLOT + half * 16;
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = *reinterpret_cast<const double2 *>(mine + i * 32);
    if (chunk == 0) x[0] = make_double2(0.0, 0.0);   // row 0: the zero ring
    __syncthreads();                             // the buffer is free again
    if (pl + (int)gridDim.x < a.npl) issue(pl + gridDim.x);
    const int pp = a.pp0 + pl;
    tri_solve<CPLX, LOGM>(x, a, pp, half, half, chunk, sh);
    const int j0 = chunk * CH, jb = j0 & (a.rows - 1);
    double2 *dst = a.dst[0] ? static_cast<double2 *>(a.dst[j0 >> lr]) + (((size_t)pp * a.rows + jb) * 2 + half)
                            : static_cast<double2 *>(a.panels) +
                                  ((((size_t)(j0 >> lr) * a.npl + pl) * a.rows + jb) * 2 + half);
#pragma unroll
    for (int i = 0; i < CH; ++i) dst[2 * i] = (j0 + i >= 1) ? x[i] : make_double2(0.0, 0.0);
  }
}

}  // namespace kfbi

namespace kfbi {

// ---------------------------------------------------------------------------
// The inverse row transform evaluated only where the trace extraction reads
// it (sweep 1 of the operator form needs the trace, not the field): for the
// stencil nodes (i, j) of one grid row j,
//   u(i, j) = 2 sum_{kx=1}^{M-1} P[kx][j] sin(pi kx i / M)
// (the DST-I of rows_inv_reg, boxsolve.py:90-93) as a direct sum over the
// column-stage output of row j.  One CTA per row with stencil nodes: the row
// and the sine table sit in shared memory, one fixed-order block reduction
// per node.  Reads each needed row once, writes nothing but the node values.
constexpr int SEVAL_E = 16;                    // row elements per thread (blockDim = M / 16)
constexpr int SEVAL_NB = 32;                   // nodes per reduction batch

template <bool CPLX>
__global__ void __launch_bounds__(512) stencil_eval_kernel(BoxArgs a, const int *__restrict__ pairs,
                                                           const int *__restrict__ pairptr,
                                                           const int *__restrict__ cols,
                                                           typename std::conditional<CPLX, double2, double>::type *vals) {
  // One CTA per row pair (2q, 2q + 1): the two rows are adjacent 32-byte
  // sectors of every strip, so they are read together.  Node entries encode
  // the column in bits 1.. and the row of the pair in bit 0.
  using T = typename std::conditional<CPLX, double2, double>::type;
  using S = Sc<T>;
  __shared__ T red[SEVAL_NB][16];
  const int M = a.m;
  const int j0 = 2 * pairs[blockIdx.x];
  const int t = threadIdx.x, nt = blockDim.x;  // nt = M / 16
  const int lane = t & 31, warp = t >> 5, nw = nt >> 5;
  T x0[SEVAL_E], x1[SEVAL_E];
#pragma unroll
  for (int e = 0; e < SEVAL_E; ++e) {
    const int kx = t + nt * e;
    if constexpr (CPLX) {
      const double2 *P2 = static_cast<const double2 *>(a.panels) + ((size_t)(kx >> 1) * a.rows + j0) * 2 + (kx & 1);
      x0[e] = P2[0];
      x1[e] = j0 + 1 < M ? P2[2] : S::zero();
    } else {
      const double *P = static_cast<const double *>(a.panels) + ((size_t)(kx >> 2) * a.rows + j0) * 4 + (kx & 3);
      x0[e] = P[0];
      x1[e] = j0 + 1 < M ? P[4] : S::zero();
    }
  }
  if (t == 0) {                                 // kx = 0: padding column
    x0[0] = S::zero();
    x1[0] = S::zero();
  }
  const int mask2 = 2 * M - 1;                  // M is a power of two
  // sin(pi n / M) for 0 <= n < 2M from the table sin(pi n / M), n < M
  auto sin_n = [&](int n) -> double { return n < M ? __ldg(&a.sinv[n]) : -__ldg(&a.sinv[n - M]); };
  const int q0 = pairptr[blockIdx.x], q1 = pairptr[blockIdx.x + 1];
  for (int qb = q0; qb < q1; qb += SEVAL_NB) {
    const int nq = min(SEVAL_NB, q1 - qb);
    for (int k = 0; k < nq; ++k) {
      const int code = cols[qb + k], i = code >> 1, odd = code & 1;
      // sin((t + nt e) pi i / M), e = 0..15: exact first two terms, then the
      // three-term recurrence s_{e+1} = 2 cos(d) s_e - s_{e-1}, d = pi nt i / M
      double sm = sin_n((t * i) & mask2);
      double s0 = sin_n(((t + nt) * i) & mask2);
      const double c2 = 2.0 * sin_n(((nt * i) + (M >> 1)) & mask2);   // 2 cos(d)
      T acc = S::rmul(odd ? x1[0] : x0[0], sm);
      acc = S::add(acc, S::rmul(odd ? x1[1] : x0[1], s0));
#pragma unroll
      for (int e = 2; e < SEVAL_E; ++e) {
        const double sn = fma(c2, s0, -sm);
        sm = s0;
        s0 = sn;
        acc = S::add(acc, S::rmul(odd ? x1[e] : x0[e], sn));
      }
      if constexpr (CPLX) {
        acc.x = warp_sum(acc.x);
        acc.y = warp_sum(acc.y);
      } else {
        acc = warp_sum(acc);
      }
      if (lane == 0) red[k][warp] = acc;
    }
    __syncthreads();
    if (t < nq) {                                 // fixed-order sum over the warps
      T s2 = S::zero();
      for (int w = 0; w < nw; ++w) s2 = S::add(s2, red[t][w]);
      vals[qb + t] = S::rmul(s2, 2.0);
    }
    __syncthreads();
  }
}

// vals[13 p + s] = node value of stencil entry (p, s) (the slab extraction layout)
template <typename T>
__global__ void __launch_bounds__(256) stencil_vals_kernel(int n, const int *__restrict__ map,
                                                           const T *__restrict__ nodevals, T *vals) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
#pragma unroll
  for (int s = 0; s < 6; ++s) vals[13 * p + s] = nodevals[map[6 * p + s]];
#pragma unroll
  for (int s = 6; s < 13; ++s) vals[13 * p + s] = Sc<T>::zero();
}

}  // namespace kfbi
