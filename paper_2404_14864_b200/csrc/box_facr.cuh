// Box solve by one level of cyclic reduction in y (FACR(1)): the same
// dirichlet-zero solve of boxsolve.py:46-94 with HALF the row transforms.
//
// With g = sign F + corrections on the interior rows and B the x operator
// (B v)_i = v_{i-1} - (4 + kappa h^2) v_i + v_{i+1} (zero ends), the 5-point
// system is u_{j-1} + B u_j + u_{j+1} = h^2 g_j.  Eliminating the odd rows,
// the even rows satisfy
//   u_{j-2} + (2 I - B^2) u_j + u_{j+2} = h^2 (g_{j-1} + g_{j+1} - B g_j)
// (u_0 = u_M = 0), which the DST along x diagonalises exactly like the full
// system: in mode kx the columns are y_{m-1} + (2 - b^2) y_m + y_{m+1} with
// b = 2 cos(pi kx / M) - 4 - kappa h^2, whose small root is r^2 (r the full
// system's root), so the tridiagonal column stage runs on M / 2 rows with
// r^2 (BoxArgs.red).  The odd rows follow from B u_j = h^2 g_j - u_{j-1} -
// u_{j+1}: one constant-coefficient tridiagonal solve along x per row
// (BoxArgs.trow, the same recurrence kernel along the row).
//
//   rows_fwd_facr : rows j-1, j, j+1 (+ corrections) -> w_j = g_{j-1} + g_{j+1}
//                   - B g_j -> DST-I(x) -> panels of the M/2 even rows
//   cols_tri (red): the even-row column systems (M/2 rows, root r^2)
//   rows_inv_reg  : panels -> DST-I(x) -> u on the even rows (row_step 2)
//   rows_odd_facr : the odd rows by x recurrences
//
// HBM traffic 5 (M-1)^2 s instead of 6 (M-1)^2 s, and half the row FFTs.
#pragma once

#include "box_reg.cuh"
#include "box_real.cuh"
#include "box_tri.cuh"

namespace kfbi {
namespace facr {

// add the sparse corrections of grid row j to a thread's elements
// n = t + m TT (m < E) (interface.py:235-238, the owner of node column i)
template <typename T, int E, int TT>
KFBI_DEV void add_row_corr(const CorrArgs<T> &c, int j, int stride, int t, T (&v)[E]) {
  if (!c.jv) return;
  const int g0 = c.row_group[j], g1 = c.row_group[j + 1];
  for (int g = g0; g < g1; ++g) {
    const int i = c.group_node[g] - j * stride;
    if (i < t || ((i - t) % TT) != 0) continue;
    const int m = (i - t) / TT;
    const T cv = group_correction<T>(c, g);
#pragma unroll
    for (int mm = 0; mm < E; ++mm)
      if (mm == m) v[mm] = Sc<T>::add(v[mm], cv);
  }
}

// The grid-row configuration of the x recurrence (one slot per CTA).
template <int LOGM>
struct CfgRow {
  static constexpr int M = 1 << LOGM;
  static constexpr int CH = M >= 1024 ? 32 : M / 32;
  static constexpr int NH = 1;
  static constexpr int NCH = M / CH;
  static constexpr int THREADS = NCH;
  static constexpr int CPW = 32;
  static constexpr int NW = NCH / 32;
  static constexpr int LCPW = 5;
  static constexpr int MINB = THREADS * 255 <= 65536 / 2 ? 2 : 1;
  static_assert(NCH >= 32 && NCH % 32 == 0 && THREADS <= 1024, "row recurrence: CTA size");
};

}  // namespace facr

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB)
rows_fwd_facr(BoxArgs a, const void *__restrict__ rhs, double sign,
              CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  using S = Sc<T>;
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T, E = reg::E;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int stride = M + 1;
  const int q = seq_index<LOGN>(seq);
  const int nseq = CPLX ? a.rows : a.rows / 2;   // a.rows = M / 2 even rows
  const bool valid = q < nseq;
  const int r0 = CPLX ? q : 2 * q;               // even-row index (row 0: the zero ring)
  const int J0 = 2 * r0;                         // grid rows 2 r0 (and 2 r0 + 2)
  // g = sign F + corrections of one grid row at this thread's elements
  auto row = [&](int j, T (&v)[E]) {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int n = t + m * TT;
      T val = S::zero();
      if (valid && j >= 1 && j <= M - 1 && n >= 1 && rhs != nullptr)
        val = S::rmul(static_cast<const T *>(rhs)[(size_t)j * stride + n], sign);
      v[m] = val;
    }
  };
  // add the corrections of grid row j (coefficient k) into component `comp`
  // of the staged sequence: distinct nodes of one row, one thread each
  // (interface.py:235-238); callers separate rows that share a slot by barriers
  auto scatter = [&](int j, int comp, double k) {
    if (!corr.jv || !valid || j < 1 || j > M - 1) return;
    const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
    for (int g = g0 + t; g < g1; g += TT) {
      const T cv = S::rmul(group_correction<T>(corr, g), k);
      const int i = corr.group_node[g] - j * stride;
      if constexpr (CPLX) {
        double2 &slot = sm.lin(i);
        slot = cadd(slot, cv);
      } else {
        double *slot = reinterpret_cast<double *>(&sm.lin(i)) + comp;
        *slot += cv;
      }
    }
  };
  // the even rows' g in shared memory (the stencil reads neighbours); the
  // odd neighbours' sum g_{j-1} + g_{j+1} is loaded right after the staging
  // for real data (its HBM latency overlaps the barrier and the corrections)
  T ga[E], gb[E];
  row(J0, ga);
  if constexpr (!CPLX) row(J0 + 2, gb);
  // (linear layout until the FFT: the stencil and the DST pre-processing
  // read shifted / mirrored windows)
  bool nzl = false;                              // any source in rows J0-1 .. J0+3 (below)
#pragma unroll
  for (int m = 0; m < E; ++m) {
    if constexpr (CPLX) {
      sm.lin(t + m * TT) = ga[m];
      nzl |= (ga[m].x != 0.0) | (ga[m].y != 0.0);
    } else {
      sm.lin(t + m * TT) = make_double2(ga[m], gb[m]);
      nzl |= (ga[m] != 0.0) | (gb[m] != 0.0);
    }
  }
  double2 os[E];
  auto load_os = [&] {
    const T *R = static_cast<const T *>(rhs);
    const bool ok = valid && rhs != nullptr;
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int n = t + m * TT;
      const bool nn = ok && n >= 1;
      auto ld = [&](int j) -> T {
        return (nn && j >= 1 && j <= M - 1) ? R[(size_t)j * stride + n] : S::zero();
      };
      if constexpr (CPLX) {
        os[m] = cscale(cadd(ld(J0 - 1), ld(J0 + 1)), sign);
      } else {
        const double mid = ld(J0 + 1);
        os[m] = make_double2((ld(J0 - 1) + mid) * sign, (mid + ld(J0 + 3)) * sign);
      }
    }
  };
  if constexpr (!CPLX) load_os();                // complex: after the corrections (registers)
  reg::seq_sync<LOGN>();
  scatter(J0, 0, 1.0);                           // the even rows' own corrections
  if constexpr (!CPLX) scatter(J0 + 2, 1, 1.0);
  reg::seq_sync<LOGN>();
  if constexpr (CPLX) load_os();
  if constexpr (C::S == 1 && C::CL == 1) {
    // rows with no source and no corrections (outside the domain's band for
    // a masked source): w = 0, whose DST is exactly 0 — write the zeros and
    // skip the stencil and the transform
#pragma unroll
    for (int m = 0; m < E; ++m) nzl |= (os[m].x != 0.0) | (os[m].y != 0.0);
    if (corr.jv && valid && t == 0) {
      for (int jj = J0 - 1; jj <= J0 + (CPLX ? 1 : 3); ++jj)
        if (jj >= 1 && jj <= M - 1 && corr.row_group[jj + 1] > corr.row_group[jj]) nzl = true;
    }
    const bool any = __syncthreads_or(nzl);
    if (a.rowz && valid && t == 0) {             // the column pass skips the loads of zero rows
      a.rowz[r0] = any ? 0 : 1;
      if constexpr (!CPLX) a.rowz[r0 + 1] = any ? 0 : 1;
    }
    if (!any) {
      if (valid && !a.rowz) {                    // (without the flags: explicit zero panels)
        const double2 z = make_double2(0.0, 0.0);
        if constexpr (!CPLX) {
#pragma unroll
          for (int kk = 0; kk < M / TT; ++kk) {
            const int i = t + kk * TT;
            *rows_fwd_dst(a, i >> 2, r0 + ((i & 3) >> 1), i & 1) = z;
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < M / TT; ++kk) {
            const int i = t + kk * TT;
            *rows_fwd_dst(a, i >> 1, r0, i & 1) = z;
          }
        }
      }
      return;
    }
  }
  // w = g_{j-1} + g_{j+1} - B g_j  (B g_j = g_{j,i-1} + g_{j,i+1} - c4 g_{j,i})
  const double2 c4 = make_double2(4.0 + a.kre * a.h2, a.kim * a.h2);
  double2 w[E];
  {
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int n = t + m * TT;
      const double2 l = n >= 1 ? sm.lin(n - 1) : make_double2(0.0, 0.0);
      const double2 rr = n + 1 <= M - 1 ? sm.lin(n + 1) : make_double2(0.0, 0.0);
      const double2 cc = sm.lin(n);
      double2 bg;                                // B g_j at n
      if constexpr (CPLX) bg = csub(cadd(l, rr), cmul(c4, cc));
      else bg = make_double2(l.x + rr.x - c4.x * cc.x, l.y + rr.y - c4.x * cc.y);
      w[m] = csub(os[m], bg);
      if (n == 0 || !valid) w[m] = make_double2(0.0, 0.0);
    }
    if (J0 == 0) {                               // even row 0: the zero ring
#pragma unroll
      for (int m = 0; m < E; ++m) w[m].x = 0.0;
      if constexpr (CPLX) {
#pragma unroll
        for (int m = 0; m < E; ++m) w[m].y = 0.0;
      }
    }
  }
  reg::seq_sync<LOGN>();                         // neighbours read before overwrite
#pragma unroll
  for (int m = 0; m < E; ++m) sm.lin(t + m * TT) = w[m];
  reg::seq_sync<LOGN>();
  // the odd rows' corrections enter w with coefficient 1; rows sharing a
  // component are separated by a barrier
  if (corr.jv) {
    if (J0 > 0) scatter(J0 - 1, 0, 1.0);
    if constexpr (!CPLX) scatter(J0 + 3, 1, 1.0);
    reg::seq_sync<LOGN>();
    if (J0 > 0) scatter(J0 + 1, 0, 1.0);
    reg::seq_sync<LOGN>();
    if constexpr (!CPLX) {
      scatter(J0 + 1, 1, 1.0);
      reg::seq_sync<LOGN>();
    }
  }
  double2 out[E];
  {
    // DST pre-processing from the linear layout (reg::pre_from_smem with
    // unswizzled reads), then the FFT and post-processing as dst_staged
    double2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
      const int j = t + m * TT;
      const double2 xj = sm.lin(j);
      const double2 xr = sm.lin((M - j) & (M - 1));   // j = 0 -> x_0 = 0
      const double s = __ldg(&a.sinv[j]);
      const double2 ap = cadd(xj, xr), dm = csub(xj, xr);
      v[m] = make_double2(fma(s, ap.x, 0.5 * dm.x), fma(s, ap.y, 0.5 * dm.y));
    }
    reg::seq_sync<LOGN>();
    reg::fft<LOGN>(v, sm, t, a.twg);
    reg::post<LOGN>(sm, t, out);
  }
  reg::seq_sync<LOGN>();
  unstage<LOGN>(sm, out, t);
  reg::seq_sync<LOGN>();
  if (valid) {
    const int ts = reg::sw(t);
    if (!CPLX) {
      const int n0t = (t & ~3) | ((t & 1) << 1);
      const int s0 = reg::sw(n0t), s1 = reg::sw(n0t + 1);
#pragma unroll
      for (int kk = 0; kk < M / TT; ++kk) {
        const int i = t + kk * TT;
        const int pp = i >> 2, part = i & 3, rw = part >> 1;
        double2 v0, v1;
        if constexpr (TT % 4 == 0) {
          v0 = sm.xc(n0t, s0, kk * TT);
          v1 = sm.xc(n0t + 1, s1, kk * TT);
        } else {
          const int n0 = 4 * pp + 2 * (part & 1);
          v0 = sm[n0];
          v1 = sm[n0 + 1];
        }
        *rows_fwd_dst(a, pp, r0 + rw, part & 1) = rw ? make_double2(v0.y, v1.y) : make_double2(v0.x, v1.x);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < M / TT; ++kk) {
        const int i = t + kk * TT;
        *rows_fwd_dst(a, i >> 1, r0, i & 1) = sm.xc(t, ts, kk * TT);
      }
    }
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

// ---------------------------------------------------------------------------
// The odd rows: B u_j = h^2 g_j - u_{j-1} - u_{j+1} along x.  Real data: two
// odd rows (j, j + 2) per CTA as the two components of a slot; complex: one.
//
// B's factored recurrences have the root rho of rho + 1/rho = 4 + kappa h^2:
// |rho| <= 2 - sqrt(3) = 0.268 whenever Re kappa >= 0 (every FACR kappa), so
// an element's influence decays below 5e-19 within W = 32 neighbours.  Each
// thread therefore solves its CH-element chunk on its own: the forward sweep
// starts W elements before the chunk and the backward sweep W elements after
// it (exact where the window reaches the ends x = 0 / x = M), with no carries
// and no scan; the boundary term at x = 0 (rho^n) needs z_1 from thread 0.
// The right-hand side is formed with coalesced loads into shared memory and
// the solution leaves the same way (padded: conflict-free chunk accesses).
constexpr int ODD_W = 32;

template <int LOGM>
struct OddCfg {
  static constexpr int M = 1 << LOGM;
  static constexpr int CH = M >= 512 ? 16 : M / 32;
  static constexpr int NT = M / CH;
};

template <int LOGM>
constexpr size_t odd_smem_bytes() {
  return ((size_t)(1 << LOGM) + (1 << LOGM) / 16 + 1) * sizeof(double2);
}

template <bool CPLX, int LOGM>
__global__ void __launch_bounds__(OddCfg<LOGM>::NT, OddCfg<LOGM>::NT <= 256 ? 2 : 1)
rows_odd_facr(BoxArgs a, const void *__restrict__ rhs, double sign,
              CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr, void *u) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  using S = Sc<T>;
  constexpr int M = OddCfg<LOGM>::M, CH = OddCfg<LOGM>::CH, NT = OddCfg<LOGM>::NT;
  extern __shared__ double2 rbuf[];              // rhs then solution, padded by one slot per 16
  __shared__ double2 z1s;
  if (a.done && *a.done) return;
  const int t = threadIdx.x;
  const int stride = M + 1;
  const int j = CPLX ? 2 * blockIdx.x + 1 : 4 * blockIdx.x + 1;   // odd row (and j + 2)
  const double h2 = a.h2;
  auto pos = [](int n) { return n + (n >> 4); };
  // a.span (the final field of a masked caller, kfbi_plan_set_field_chunks):
  // only the chunks [c_lo, c_hi] of this row (pair) are needed; loads outside
  // their windows and the x = 0 boundary term (rho^n z_1, n >= 64: below the
  // rounding of y) are skipped
  int c_lo = 0, c_hi = NT - 1, nlo = 0, nhi = M;
  if (a.span) {
    int2 sp = a.span[(j - 1) >> 1];
    if constexpr (!CPLX) {                     // rows j and j + 2: the union of the ranges
      const int2 s2 = a.span[(j + 1) >> 1];
      const bool e1 = sp.x <= sp.y;
      if (s2.x <= s2.y) sp = e1 ? make_int2(min(sp.x, s2.x), max(sp.y, s2.y)) : s2;
    }
    if (sp.x > sp.y) return;                     // nothing of this row (pair) is read
    c_lo = sp.x;
    c_hi = sp.y;
    nlo = CH * c_lo - ODD_W - 1;
    nhi = CH * (c_hi + 1) + ODD_W;
  }
  // rhs_n = h^2 g_j - u_{j-1} - u_{j+1} (u_0 = u_M = 0), coalesced over n = t + NT e
  auto form = [&](int jj, int comp) {
    const T *U = static_cast<const T *>(u);
    const T *Fr = static_cast<const T *>(rhs) + (size_t)jj * stride;
    const T *Ul = U + (size_t)(jj - 1) * stride, *Uh = U + (size_t)(jj + 1) * stride;
    const bool hasl = jj - 1 >= 1, hash = jj + 1 <= M - 1;
    T f[CH], l[CH], hv[CH];                      // every load in flight before any use
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int n = t + NT * e;
      const bool w = n >= nlo && n <= nhi;
      f[e] = (rhs && w) ? Fr[n] : S::zero();
      l[e] = (hasl && w) ? Ul[n] : S::zero();
      hv[e] = (hash && w) ? Uh[n] : S::zero();
    }
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int n = t + NT * e;
      T val = S::sub(S::sub(S::rmul(f[e], sign * h2), l[e]), hv[e]);
      if (n == 0) val = S::zero();
      if constexpr (CPLX) rbuf[pos(n)] = val;
      else reinterpret_cast<double *>(&rbuf[pos(n)])[comp] = val;
    }
  };
  if constexpr (CPLX) {
    form(j, 0);
  } else {
    // both rows per slot in one 16-byte store (8-byte stores into 16-byte
    // slots were 2-way bank conflicts): rows j, j + 2 share row j + 1, so
    // five row loads per element, eight elements in flight
    const double *R = static_cast<const double *>(rhs);
    const double *U = static_cast<const double *>(u);
    const double *F0 = R + (size_t)j * stride, *F1 = F0 + 2 * (size_t)stride;
    const double *Ua = U + (size_t)(j - 1) * stride;     // u_{j-1}
    const double *Ub = Ua + 2 * (size_t)stride;          // u_{j+1}
    const double *Uc = Ub + 2 * (size_t)stride;          // u_{j+3}
    const bool ha = j - 1 >= 1, hc = j + 3 <= M - 1;
    constexpr int HB = CH >= 8 ? 8 : CH;
#pragma unroll
    for (int e0 = 0; e0 < CH; e0 += HB) {
      double f0[HB], f1[HB], la[HB], lb[HB], lc[HB];
#pragma unroll
      for (int e = 0; e < HB; ++e) {
        const int n = t + NT * (e0 + e);
        const bool w = n >= nlo && n <= nhi;
        f0[e] = (rhs && w) ? F0[n] : 0.0;
        f1[e] = (rhs && w) ? F1[n] : 0.0;
        la[e] = (ha && w) ? Ua[n] : 0.0;
        lb[e] = w ? Ub[n] : 0.0;
        lc[e] = (hc && w) ? Uc[n] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < HB; ++e) {
        const int n = t + NT * (e0 + e);
        const double v0 = f0[e] * (sign * h2) - la[e] - lb[e];
        const double v1 = f1[e] * (sign * h2) - lb[e] - lc[e];
        rbuf[pos(n)] = n == 0 ? make_double2(0.0, 0.0) : make_double2(v0, v1);
      }
    }
  }
  __syncthreads();
  if (corr.jv) {                                 // corrections of the row(s), h^2 scaled:
    for (int k2 = 0; k2 < (CPLX ? 1 : 2); ++k2) {  // distinct nodes, one thread each
      const int jj = j + 2 * k2;
      const int g0 = corr.row_group[jj], g1 = corr.row_group[jj + 1];
      for (int g = g0 + t; g < g1; g += NT) {
        const int i = corr.group_node[g] - jj * stride;
        const T cv = S::rmul(group_correction<T>(corr, g), h2);
        if constexpr (CPLX) rbuf[pos(i)] = cadd(rbuf[pos(i)], cv);
        else reinterpret_cast<double *>(&rbuf[pos(i)])[k2] += cv;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // this thread's chunk [s, s + CH) with windows
  const double2 r = tri::root_cplx(make_double2(a.tb_re, a.tb_im));   // rho (imag 0 for real kappa)
  double2 rr;                                    // the slot multiplier
  if constexpr (CPLX) rr = r;
  else rr = make_double2(r.x, r.x);
  const int s0 = t * CH;
  const int lo = s0 - ODD_W < 1 ? 1 : s0 - ODD_W;               // exact start at x = 1 (v_0 = 0)
  const int hi = s0 + CH + ODD_W > M - 1 ? M - 1 : s0 + CH + ODD_W;  // exact end at x = M - 1 (z_M = 0)
  // forward v_n = rho v_{n-1} - rhs_n over [lo, hi]: v kept on the chunk; after
  // it only z at the chunk end, z_end = sum_{n >= end} rho^{n - end} v_n
  const bool act = t >= c_lo && t <= c_hi;       // (always, without a span)
  double2 zch[CH];
  double2 v = make_double2(0.0, 0.0);
#pragma unroll 8
  for (int n = lo; n < (act ? s0 : lo); ++n) v = tri::mad<CPLX>(rr, v, cneg(rbuf[pos(n)]));
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    const int n = s0 + e;
    if (n >= 1) v = tri::mad<CPLX>(rr, v, cneg(rbuf[pos(n)]));
    zch[e] = v;                                  // n = 0: v_0 = 0
  }
  double2 z = make_double2(0.0, 0.0), pw1 = tri::one<CPLX>();
#pragma unroll 8
  for (int n = s0 + CH; n <= (act ? hi : s0); ++n) {
    v = tri::mad<CPLX>(rr, v, cneg(rbuf[pos(n)]));
    z = tri::mad<CPLX>(pw1, v, z);
    pw1 = tri::mul<CPLX>(pw1, rr);
  }
  // backward z_n = rho z_{n+1} + v_n through the chunk (in place)
#pragma unroll
  for (int e = CH - 1; e >= 0; --e) {
    z = tri::mad<CPLX>(rr, z, zch[e]);
    zch[e] = z;
  }
  if (t == 0) z1s = zch[CH > 1 ? 1 : 0];          // z_1 (CH >= 2 always here)
  __syncthreads();                               // rhs reads done; z_1 visible
  // y_n = rho z_n + B rho^n, B = -rho^2 z_1 (rho^{2M} terms < 1e-300)
  const double2 Bc = a.span ? make_double2(0.0, 0.0) : cneg(tri::mul<CPLX>(tri::mul<CPLX>(rr, rr), z1s));
  double2 pw = tri::pw<CPLX>(rr, s0);            // rho^n
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    const double2 y = tri::mad<CPLX>(Bc, pw, tri::mul<CPLX>(rr, zch[e]));
    rbuf[pos(s0 + e)] = y;
    pw = tri::mul<CPLX>(pw, rr);
  }
  __syncthreads();
  T *U = static_cast<T *>(u);
  const int olo = a.span ? CH * c_lo : 0, ohi = a.span ? CH * (c_hi + 1) - 1 : M;
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    const int n = t + NT * e;
    if (n < olo || n > ohi) continue;
    const double2 y = rbuf[pos(n)];
    if constexpr (CPLX) {
      U[(size_t)j * stride + n] = n >= 1 ? y : S::zero();
    } else {
      U[(size_t)j * stride + n] = n >= 1 ? y.x : 0.0;
      U[(size_t)(j + 2) * stride + n] = n >= 1 ? y.y : 0.0;
    }
  }
  if (a.span) return;                            // (ring column / row: exterior, never read)
  if (t == 0) {                                  // x = M: the zero ring column
    U[(size_t)j * stride + M] = S::zero();
    if constexpr (!CPLX) U[(size_t)(j + 2) * stride + M] = S::zero();
  }
  // the zero ring row M, written by the CTA of the last odd row
  const int last = CPLX ? M - 1 : M - 3;
  if (j == last)
    for (int i = t; i <= M; i += NT) U[(size_t)M * stride + i] = S::zero();
}

}  // namespace kfbi

namespace kfbi {

// ---------------------------------------------------------------------------
// The odd rows of a trace-only first sweep: only the 16-element chunks that
// hold six-point stencil nodes (BoxArgs.oc_list, built with the geometry).
// One warp per chunk: the lanes stage the chunk's right-hand side over its
// windows [s0 - W, s0 + 16 + W] (h^2 g - u_{j-1} - u_{j+1} + corrections, as
// rows_odd_facr forms it), then lane 0 runs exactly rows_odd_facr's
// recurrences for that chunk.  The chunks never reach x = 0, where the one
// boundary term of the full row lives (rho^n z_1 with n >= 64: below the
// rounding of y).
constexpr int OS_WARPS = 4;
template <bool CPLX, int LOGM>
__global__ void __launch_bounds__(OS_WARPS * 32)
rows_odd_facr_sparse(BoxArgs a, const void *__restrict__ rhs, double sign,
                     CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr, void *u) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  using S = Sc<T>;
  constexpr int M = 1 << LOGM, CH = 16, WIN = CH + 2 * ODD_W + 1;
  __shared__ double2 win[OS_WARPS][WIN];
  if (a.done && *a.done) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q = blockIdx.x * OS_WARPS + w;
  if (q >= a.n_oc) return;
  const int2 jc = a.oc_list[q];
  const int j = jc.x, s0 = CH * jc.y;
  const int stride = M + 1;
  const int lo = s0 - ODD_W, hi = s0 + CH + ODD_W;     // interior windows (checked at build)
  const double h2 = a.h2;
  const T *F = static_cast<const T *>(rhs);
  const T *U = static_cast<const T *>(u);
  double2 *wb = win[w];
  for (int k = lane; k <= hi - lo; k += 32) {
    const int n = lo + k;
    const T f = rhs ? F[(size_t)j * stride + n] : S::zero();
    const T l = U[(size_t)(j - 1) * stride + n];
    const T h = j + 1 <= M - 1 ? U[(size_t)(j + 1) * stride + n] : S::zero();
    const T val = S::sub(S::sub(S::rmul(f, sign * h2), l), h);
    if constexpr (CPLX) wb[k] = val;
    else wb[k] = make_double2(val, 0.0);
  }
  __syncwarp();
  if (corr.jv) {                                 // the row's corrections inside the window
    const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
    for (int g = g0 + lane; g < g1; g += 32) {
      const int i = corr.group_node[g] - j * stride;
      if (i >= lo && i <= hi) {
        const T cv = S::rmul(group_correction<T>(corr, g), h2);
        if constexpr (CPLX) wb[i - lo] = cadd(wb[i - lo], cv);
        else wb[i - lo].x += cv;
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    const double2 r = tri::root_cplx(make_double2(a.tb_re, a.tb_im));
    double2 rr;
    if constexpr (CPLX) rr = r;
    else rr = make_double2(r.x, r.x);
    auto x = [&](int n) { return wb[n - lo]; };
    double2 zch[CH];
    double2 v = make_double2(0.0, 0.0);
    for (int n = lo; n < s0; ++n) v = tri::mad<CPLX>(rr, v, cneg(x(n)));
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      v = tri::mad<CPLX>(rr, v, cneg(x(s0 + e)));
      zch[e] = v;
    }
    double2 z = make_double2(0.0, 0.0), pw1 = tri::one<CPLX>();
    for (int n = s0 + CH; n <= hi; ++n) {
      v = tri::mad<CPLX>(rr, v, cneg(x(n)));
      z = tri::mad<CPLX>(pw1, v, z);
      pw1 = tri::mul<CPLX>(pw1, rr);
    }
#pragma unroll
    for (int e = CH - 1; e >= 0; --e) {
      z = tri::mad<CPLX>(rr, z, zch[e]);
      zch[e] = z;
    }
    T *Uo = static_cast<T *>(u) + (size_t)j * stride;
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const double2 y = tri::mul<CPLX>(rr, zch[e]);
      if constexpr (CPLX) Uo[s0 + e] = y;
      else Uo[s0 + e] = y.x;
    }
  }
}

// ---------------------------------------------------------------------------
// FACR(1) for REAL data at M = 16384 on the one-real-row-per-CTA engine of
// box_real.cuh (length-8192 complex FFT with the real split).

// even grid row j = 2 r0 (r0 = blockIdx.x, reduced row): w_j = g_{j-1} +
// g_{j+1} - B g_j, staged as pairs (x_2q, x_2q+1), then the real DST-I
template <int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN - 1>::CTA_T, 1)
rows_fwd_facr_real(BoxArgs a, const double *__restrict__ rhs, double sign, CorrArgs<double> corr) {
  constexpr int LOGL = LOGN - 1;
  using C = reg::Cfg<LOGL>;
  static_assert(C::S == 1 && C::CL == 1, "one sequence per CTA");
  constexpr int M = 1 << LOGN, L = C::N, TT = C::T, E = reg::E;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGL> sm = reg::make_view<LOGL>(smem, seq, t);
  const int stride = M + 1;
  const int r0 = blockIdx.x;                     // reduced (even) row
  const int j = 2 * r0;                          // grid row
  auto ldrow = [&](int jj, int q, double &x0, double &x1) {
    x0 = x1 = 0.0;
    if (jj >= 1 && jj <= M - 1 && rhs != nullptr) {
      const double *row = rhs + (size_t)jj * stride;
      if (q >= 1) x0 = row[2 * q] * sign;
      x1 = row[2 * q + 1] * sign;
    }
  };
  auto scatter = [&](int jj) {                   // corrections of grid row jj into the staged pairs
    if (!corr.jv || jj < 1 || jj > M - 1) return;
    const int g0 = corr.row_group[jj], g1 = corr.row_group[jj + 1];
    for (int g = g0 + t; g < g1; g += TT) {
      const double cv = group_correction<double>(corr, g);
      const int i = corr.group_node[g] - jj * stride;
      reinterpret_cast<double *>(&sm[i >> 1])[i & 1] += cv;
    }
  };
  {
    double2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) ldrow(j, t + m * TT, v[m].x, v[m].y);
    stage<LOGL>(sm, v, t);
  }
  reg::seq_sync<LOGL>();
  scatter(j);
  reg::seq_sync<LOGL>();
  const double c4 = 4.0 + a.kre * a.h2;
  double2 w[E];
#pragma unroll
  for (int m = 0; m < E; ++m) {
    const int q = t + m * TT;                    // elements 2q, 2q + 1
    double l0, l1, h0, h1;
    ldrow(j - 1, q, l0, l1);
    ldrow(j + 1, q, h0, h1);
    const double2 c = sm[q];
    const double left = q >= 1 ? sm[q - 1].y : 0.0;           // g[2q - 1]
    const double right = q + 1 < L ? sm[q + 1].x : 0.0;       // g[2q + 2] (g[M] = 0)
    const double b0 = left + c.y - c4 * c.x;                  // (B g)[2q]
    const double b1 = c.x + right - c4 * c.y;                 // (B g)[2q + 1]
    w[m] = make_double2(q >= 1 ? l0 + h0 - b0 : 0.0, l1 + h1 - b1);
    if (j == 0) w[m] = make_double2(0.0, 0.0);
  }
  if (a.rowz) {
    // no source and no corrections in rows j-1 .. j+1 (outside the domain's
    // band for a masked source): the DST of w = 0 is exactly 0, the column
    // pass skips the row (rowz) and no panel is written
    bool nzl = false;
#pragma unroll
    for (int m = 0; m < E; ++m) nzl |= (w[m].x != 0.0) | (w[m].y != 0.0);
    if (corr.jv && t == 0 && j > 0)
      for (int jj = j - 1; jj <= j + 1; jj += 2)
        if (jj <= M - 1 && corr.row_group[jj + 1] > corr.row_group[jj]) nzl = true;
    const bool any = __syncthreads_or(nzl);
    if (t == 0) a.rowz[r0] = any ? 0 : 1;
    if (!any) return;
  }
  reg::seq_sync<LOGL>();
  stage<LOGL>(sm, w, t);
  reg::seq_sync<LOGL>();
  if (j > 0) {                                   // odd rows' corrections, one row per barrier
    scatter(j - 1);
    reg::seq_sync<LOGL>();
    scatter(j + 1);
    reg::seq_sync<LOGL>();
  }
  double2 out[E];
  realdst::dst_staged<LOGL>(sm, t, a, out);
  reg::seq_sync<LOGL>();
  unstage<LOGL>(sm, out, t);
  reg::seq_sync<LOGL>();
  for (int i = t; i < L; i += TT) *rows_fwd_dst(a, i >> 1, r0, i & 1) = sm[i];
}

// odd grid row j (one real row per CTA): B u_j = h^2 g_j - u_{j-1} - u_{j+1}
// by windowed recurrences (|rho| <= 0.268), as rows_odd_facr
template <int LOGM>
constexpr size_t odd1_smem_bytes() {
  return ((size_t)(1 << LOGM) + (1 << LOGM) / 16 + 1) * sizeof(double);
}

template <int LOGM>
__global__ void __launch_bounds__(1024, 1)
rows_odd_facr_real1(BoxArgs a, const double *__restrict__ rhs, double sign, CorrArgs<double> corr,
                    double *u) {
  constexpr int M = 1 << LOGM, CH = 16, NT = M / CH;
  static_assert(NT <= 1024, "one chunk of 16 per thread");
  extern __shared__ double rb1[];
  __shared__ double z1s;
  if (a.done && *a.done) return;
  const int t = threadIdx.x;
  const int stride = M + 1;
  const int j = 2 * blockIdx.x + 1;
  const double h2 = a.h2;
  auto pos = [](int n) { return n + (n >> 4); };
  {
    const double *Fr = rhs + (size_t)j * stride;
    const double *Ul = u + (size_t)(j - 1) * stride, *Uh = u + (size_t)(j + 1) * stride;
    const bool hasl = j - 1 >= 1, hash = j + 1 <= M - 1;
    double f[CH], l[CH], hv[CH];
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int n = t + NT * e;
      f[e] = rhs ? Fr[n] : 0.0;
      l[e] = hasl ? Ul[n] : 0.0;
      hv[e] = hash ? Uh[n] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int n = t + NT * e;
      rb1[pos(n)] = n >= 1 ? f[e] * (sign * h2) - l[e] - hv[e] : 0.0;
    }
  }
  __syncthreads();
  if (corr.jv) {
    const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
    for (int g = g0 + t; g < g1; g += NT) {
      const int i = corr.group_node[g] - j * stride;
      rb1[pos(i)] += group_correction<double>(corr, g) * h2;
    }
    __syncthreads();
  }
  const double r = tri::root_real(a.tb_re);
  const int s0 = t * CH;
  const int lo = s0 - ODD_W < 1 ? 1 : s0 - ODD_W;
  const int hi = s0 + CH + ODD_W > M - 1 ? M - 1 : s0 + CH + ODD_W;
  double zc[CH];
  double v = 0.0;
#pragma unroll 8
  for (int n = lo; n < s0; ++n) v = fma(r, v, -rb1[pos(n)]);
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    const int n = s0 + e;
    if (n >= 1) v = fma(r, v, -rb1[pos(n)]);
    zc[e] = v;
  }
  double z = 0.0, pw1 = 1.0;
#pragma unroll 8
  for (int n = s0 + CH; n <= hi; ++n) {
    v = fma(r, v, -rb1[pos(n)]);
    z = fma(pw1, v, z);
    pw1 *= r;
  }
#pragma unroll
  for (int e = CH - 1; e >= 0; --e) {
    z = fma(r, z, zc[e]);
    zc[e] = z;
  }
  if (t == 0) z1s = zc[1];
  __syncthreads();
  const double Bc = -(r * r) * z1s;
  double pw = 1.0;
  for (int k = 0; k < s0 && pw != 0.0; ++k) pw *= r;   // r^s0 (underflows to 0 quickly)
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    rb1[pos(s0 + e)] = fma(Bc, pw, r * zc[e]);
    pw *= r;
  }
  __syncthreads();
  double *urow = u + (size_t)j * stride;
#pragma unroll
  for (int e = 0; e < CH; ++e) {
    const int n = t + NT * e;
    urow[n] = n >= 1 ? rb1[pos(n)] : 0.0;
  }
  if (t == 0) urow[M] = 0.0;
  if (j == M - 1)
    for (int i = t; i <= M; i += NT) u[(size_t)M * stride + i] = 0.0;
}

}  // namespace kfbi
