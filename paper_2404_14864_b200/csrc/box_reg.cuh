// Box solve (Delta_h - kappa) u = rhs, dirichlet-zero closure
// (BoxSolver.solve, boxsolve.py:46-94) on the register DST-I engine
// (dst_reg.cuh), three HBM passes:
//
//   rows_fwd_reg : rhs rows (+ the sparse jump corrections of those rows,
//                  interface.py:235-238 / bvp.py:319) -> DST-I along x -> panels
//   cols_reg     : panel column -> DST-I along y -> / (lam_p + lam_q - kappa)
//                  / (4 M^2) -> DST-I along y -> panel column (in place)
//   rows_inv_reg : panels -> DST-I along x -> u rows with the exact zero ring
//
// Panels (the intermediate spectrum): 32-byte column strips indexed by the
// spectral x index kx (column 0 is padding) and the row / spectral y index j
// (row 0 is the zero ring).  Real: panel pp holds kx = 4pp..4pp+3,
// P[(pp*R + r)*4 + w]; complex: kx = 2pp..2pp+1, P2[(pp*R + r)*2 + w], with
// r the row within the slab of R rows (R = M on one GPU).  A column pass
// reads one 32-byte-wide strip per panel (two CTAs per strip, one per
// 16-byte half); a row pair (2q, 2q+1) of a real panel is one contiguous
// 64-byte chunk.  All global traffic goes through the shared-memory staging
// buffer so that consecutive lanes touch consecutive 16-byte pieces.
//
// Slab decomposition (BoxArgs rows/row0/pp0/npl): the row passes of rank g
// touch only its rows, the column pass only its panels, and the two
// all-to-all transposes between them (NCCL, dist.py) move whole contiguous
// [panel range][rows] blocks, so no pack / unpack pass exists.
//
// One CTA = 256 threads = 256*16 complex elements in registers: one length-
// 4096 sequence, or 4096/N shorter ones.  Real rows/columns are packed two
// per complex sequence.
#pragma once

#include "box_kernels.cuh"
#include "dst_reg.cuh"

namespace kfbi {

// stage x (natural order) into the sequence's smem
template <int LOGN>
KFBI_DEV void stage(const reg::View<LOGN> &sm, const double2 (&v)[reg::E], int t) {
#pragma unroll
  for (int m = 0; m < reg::E; ++m) sm.xc(t, reg::sw(t), m * reg::Cfg<LOGN>::T) = v[m];
}

// write out[c] (index 16 t + c) to the sequence's smem in natural order
template <int LOGN>
KFBI_DEV void unstage(const reg::View<LOGN> &sm, const double2 (&out)[reg::E], int t) {
#pragma unroll
  for (int c = 0; c < reg::E; ++c) sm.xc(reg::E * t, reg::sw(reg::E * t), c) = out[c];
}

// x staged in sm -> C = DST-I(x) in out[c] (index 16 t + c).  Entry: staged
// data visible (after a barrier).  Exit: sm may still be read by other
// threads (barrier needed before the next write).
template <int LOGN>
KFBI_DEV void dst_staged(const reg::View<LOGN> &sm, int t, const BoxArgs &a, double2 (&out)[reg::E]) {
  double2 v[reg::E];
  reg::pre_from_smem<LOGN>(v, sm, t, a.sinv);
  reg::seq_sync<LOGN>();
  reg::fft<LOGN>(v, sm, t, a.twg);
  reg::post<LOGN>(sm, t, out);
}

// sequence index of the calling thread's sequence
template <int LOGN>
KFBI_DEV int seq_index(int seq) {
  using C = reg::Cfg<LOGN>;
  if constexpr (C::CL == 1) return blockIdx.x * C::S + seq;
  else return blockIdx.x / C::CL;
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB)
rows_fwd_reg(BoxArgs a, const void *__restrict__ rhs, double sign,
             CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int stride = M + 1;
  const int q = seq_index<LOGN>(seq);
  const int nseq = CPLX ? a.rows : a.rows / 2;
  const bool valid = q < nseq;
  const int r0 = CPLX ? q : 2 * q;               // slab row of the sequence
  const int j0 = a.row0 + r0;                    // grid row (row 0: zero ring)

  double2 v[reg::E];
#pragma unroll
  for (int m = 0; m < reg::E; ++m) {
    const int n = t + m * TT;
    v[m] = make_double2(0.0, 0.0);
    if (valid && n >= 1 && rhs != nullptr) {
      if (CPLX) {
        if (j0 >= 1) v[m] = static_cast<const double2 *>(rhs)[(size_t)r0 * stride + n];
      } else {
        const double *r = static_cast<const double *>(rhs);
        if (j0 >= 1) v[m].x = r[(size_t)r0 * stride + n];
        v[m].y = r[(size_t)(r0 + 1) * stride + n];
      }
    }
  }
#pragma unroll
  for (int m = 0; m < reg::E; ++m) v[m] = cscale(v[m], sign);
  stage<LOGN>(sm, v, t);
  if (corr.jv) {
    reg::seq_sync<LOGN>();
    if (valid) {
      const int nrows = CPLX ? 1 : 2;
      for (int qq = (j0 == 0); qq < nrows; ++qq) {
        const int j = j0 + qq;
        const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
        for (int g = g0 + t; g < g1; g += TT) {
          const T cv = group_correction<T>(corr, g);
          const int i = corr.group_node[g] - j * stride;
          if constexpr (CPLX) {
            double2 &slot = sm[i];
            slot = cadd(slot, cv);
          } else {
            double *slot = reinterpret_cast<double *>(&sm[i]) + qq;
            *slot += cv;
          }
        }
      }
    }
  }
  reg::seq_sync<LOGN>();
  double2 out[reg::E];
  dst_staged<LOGN>(sm, t, a, out);
  reg::seq_sync<LOGN>();
  unstage<LOGN>(sm, out, t);
  reg::seq_sync<LOGN>();
  if (valid) {
    // panel stores: consecutive lanes write consecutive 16-byte pieces of a
    // panel's (row j0, row j0+1) 64-byte chunk (real) / 32-byte row (complex)
    // (i = t + kk TT: the shared-memory slots are t's plus a constant)
    const int ts = reg::sw(t);
    if (!CPLX) {
      const int n0t = (t & ~3) | ((t & 1) << 1);   // slot pair of piece t
      const int s0 = reg::sw(n0t), s1 = reg::sw(n0t + 1);
#pragma unroll
      for (int kk = 0; kk < M / TT; ++kk) {      // M/4 panels x 4 pieces
        const int i = t + kk * TT;
        const int pp = i >> 2, part = i & 3, row = part >> 1;
        // n0(i) = n0(t) + kk TT needs TT % 4 == 0 (M >= 64); else the plain index
        double2 v0, v1;
        if constexpr (TT % 4 == 0) {
          v0 = sm.xc(n0t, s0, kk * TT);
          v1 = sm.xc(n0t + 1, s1, kk * TT);
        } else {
          const int n0 = 4 * pp + 2 * (part & 1);
          v0 = sm[n0];
          v1 = sm[n0 + 1];
        }
        *rows_fwd_dst(a, pp, r0 + row, part & 1) =
            row ? make_double2(v0.y, v1.y) : make_double2(v0.x, v1.x);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < M / TT; ++kk) {      // M/2 panels x 2 pieces
        const int i = t + kk * TT;
        *rows_fwd_dst(a, i >> 1, r0, i & 1) = sm.xc(t, ts, kk * TT);
      }
    }
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();   // keep the cluster's smem alive
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB) cols_reg(BoxArgs a) {
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  const int q = seq_index<LOGN>(seq);
  const int nseq = 2 * a.npl;                    // half panels of this rank
  const bool valid = q < nseq;
  const int pl = q >> 1, half = q & 1;
  const int pp = a.pp0 + pl;                     // global panel
  // row j of the strip lives in rank block j / R (R = a.rows, a power of two)
  const int lr = 31 - __clz(a.rows);
  double2 *P2 = static_cast<double2 *>(a.panels);
  auto at = [&](int j) -> double2 & {
    const size_t blk = (size_t)(j >> lr) * a.npl + pl;
    return P2[(blk * a.rows + (j & (a.rows - 1))) * 2 + half];
  };
  // result element j: in place, or into the row-pass buffer of row j's owner
  auto out_at = [&](int j) -> double2 & {
    if (!a.dst[0]) return at(j);
    return static_cast<double2 *>(a.dst[j >> lr])[((size_t)pp * a.rows + (j & (a.rows - 1))) * 2 + half];
  };

  double2 v[reg::E];
  double2 out[reg::E];
  if constexpr (C::CL == 1) {
    // DST-I pre-processing straight from global memory: element n and its
    // mirror M - n (the same strip, an L2 hit for one of the two loads)
    // instead of staging the column through shared memory
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double2 x[reg::E / 2], xr[reg::E / 2];
#pragma unroll
      for (int mm = 0; mm < reg::E / 2; ++mm) {
        const int n = t + (h * (reg::E / 2) + mm) * TT;
        x[mm] = (valid && n >= 1) ? at(n) : make_double2(0.0, 0.0);
        xr[mm] = (valid && n >= 1) ? at(M - n) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int mm = 0; mm < reg::E / 2; ++mm) {
        const int n = t + (h * (reg::E / 2) + mm) * TT;
        const double sj = __ldg(&a.sinv[n]);
        const double2 ad = cadd(x[mm], xr[mm]), df = csub(x[mm], xr[mm]);
        v[h * (reg::E / 2) + mm] = make_double2(fma(sj, ad.x, 0.5 * df.x), fma(sj, ad.y, 0.5 * df.y));
      }
    }
    reg::fft<LOGN>(v, sm, t, a.twg);
    reg::post<LOGN>(sm, t, out);
  } else {
#pragma unroll
    for (int m = 0; m < reg::E; ++m) {
      const int n = t + m * TT;
      v[m] = (valid && n >= 1) ? at(n) : make_double2(0.0, 0.0);
    }
    stage<LOGN>(sm, v, t);
    reg::seq_sync<LOGN>();
    dst_staged<LOGN>(sm, t, a, out);
  }

  // spectral division (boxsolve.py:74-76): (v / (lam_p + lam_q - kappa)) / (4 M^2)
#pragma unroll
  for (int c = 0; c < reg::E; ++c) {
    const int p = reg::E * t + c;
    const double lp = a.lam[p];
    if (!CPLX) {
      const int kx = valid ? 4 * pp + 2 * half : 0;   // idle sequences stay in bounds
      const double da = (lp + a.lam[kx]) - a.kre;
      const double db = (lp + a.lam[kx + 1]) - a.kre;
      out[c] = make_double2((out[c].x / da) * a.inv4m2, (out[c].y / db) * a.inv4m2);
    } else {
      const int kx = valid ? 2 * pp + half : 0;
      const double2 d = make_double2((lp + a.lam[kx]) - a.kre, -a.kim);
      out[c] = cscale(cdiv(out[c], d), a.inv4m2);
    }
  }
  if (t == 0) out[0] = make_double2(0.0, 0.0);   // x_0 = 0 for the second transform
  reg::seq_sync<LOGN>();
  if constexpr (C::CL == 1 && TT >= 32) {
    // second transform in transposed form: its input is the first one's
    // output layout and its output the column's row layout
    reg::dst_transposed<LOGN>(sm, t, out, v, a.twg, a.sinv);
    if (valid)
#pragma unroll
      for (int m = 0; m < reg::E; ++m) {
        const int n = t + m * TT;
        out_at(n) = n >= 1 ? v[m] : make_double2(0.0, 0.0);   // row 0: zero ring
      }
  } else {
    unstage<LOGN>(sm, out, t);
    reg::seq_sync<LOGN>();
    dst_staged<LOGN>(sm, t, a, out);
    reg::seq_sync<LOGN>();
    unstage<LOGN>(sm, out, t);
    reg::seq_sync<LOGN>();
    if (valid)
#pragma unroll
      for (int kk = 0; kk < M / TT; ++kk) out_at(t + kk * TT) = sm.xc(t, reg::sw(t), kk * TT);
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

// ---------------------------------------------------------------------------
template <bool CPLX, int LOGN>
__global__ void __launch_bounds__(reg::Cfg<LOGN>::CTA_T, reg::Cfg<LOGN>::MINB)
rows_inv_reg(BoxArgs a, void *__restrict__ u) {
  using C = reg::Cfg<LOGN>;
  constexpr int M = C::N, TT = C::T;
  extern __shared__ double2 smem[];
  if (a.done && *a.done) return;
  int seq, t;
  const reg::View<LOGN> sm = reg::make_view<LOGN>(smem, seq, t);
  // staging slot of element n: linear for one-CTA sequences (see View::lin)
  auto stg = [&](int n) -> double2 & {
    if constexpr (C::CL == 1) return sm.lin(n);
    else return sm[n];
  };
  const int stride = M + 1;
  const int q = seq_index<LOGN>(seq);
  const int nseq = CPLX ? a.rows : a.rows / 2;
  const bool valid = q < nseq;
  const int r0 = CPLX ? q : 2 * q;               // slab row of the sequence
  const int j0 = a.row0 + r0;                    // grid row (row 0: zero ring)
  const size_t R = a.rows;
  // rows nobody reads (trace-only / masked FACR solves, outside the domain's
  // rows): the whole sequence is skipped (one sequence per CTA only)
  if constexpr (C::S == 1 && C::CL == 1) {
    if (a.row_need && valid && !a.row_need[r0] && (CPLX || !a.row_need[r0 + 1])) return;
  }

  const double2 *P2 = static_cast<const double2 *>(a.panels);
  if (!CPLX) {
    // lanes read consecutive 16-byte pieces of each panel's (r0, r0+1)
    // 64-byte chunk and scatter them into the .x / .y halves of the slots
    double2 v[reg::E];
#pragma unroll
    for (int m = 0; m < reg::E; ++m) {
      const int i = t + m * TT, pp = i >> 2, part = i & 3, row = part >> 1;
      v[m] = valid ? P2[(pp * R + r0 + row) * 2 + (part & 1)] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int m = 0; m < reg::E; ++m) {
      const int i = t + m * TT, pp = i >> 2, part = i & 3, row = part >> 1;
      const int n0 = 4 * pp + 2 * (part & 1);
      double *s0 = reinterpret_cast<double *>(&stg(n0)) + row;
      double *s1 = reinterpret_cast<double *>(&stg(n0 + 1)) + row;
      *s0 = n0 == 0 ? 0.0 : v[m].x;            // x_0 = 0
      *s1 = v[m].y;
    }
  } else {
    double2 v[reg::E];
#pragma unroll
    for (int m = 0; m < reg::E; ++m) {
      const int n = t + m * TT;
      v[m] = (valid && n >= 1) ? P2[((n >> 1) * R + r0) * 2 + (n & 1)] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int m = 0; m < reg::E; ++m) stg(t + m * TT) = v[m];
  }
  reg::seq_sync<LOGN>();
  double2 out[reg::E];
  if constexpr (C::CL == 1) {
    // pre-processing from the linear staging (mirror reads without the
    // swizzle-group conflicts), then the FFT and post-processing
    double2 v[reg::E];
#pragma unroll
    for (int m = 0; m < reg::E; ++m) {
      const int j = t + m * TT;
      const double2 xj = sm.lin(j);
      const double2 xr = sm.lin((M - j) & (M - 1));
      const double s = __ldg(&a.sinv[j]);
      const double2 ap = cadd(xj, xr), dm = csub(xj, xr);
      v[m] = make_double2(fma(s, ap.x, 0.5 * dm.x), fma(s, ap.y, 0.5 * dm.y));
    }
    reg::seq_sync<LOGN>();
    reg::fft<LOGN>(v, sm, t, a.twg);
    reg::post<LOGN>(sm, t, out);
  } else {
    dst_staged<LOGN>(sm, t, a, out);
  }
  reg::seq_sync<LOGN>();
  unstage<LOGN>(sm, out, t);
  reg::seq_sync<LOGN>();
  if (valid) {
    // coalesced row stores with the zero ring (boxsolve.py:90-93); grid row
    // 0 comes out of the transforms as exact zeros (its input is zero)
    const bool last = a.ring_end && q == nseq - 1;   // also write ring row M
    if (!CPLX) {
      double *U = static_cast<double *>(u);
      double *u0 = U + (size_t)r0 * a.row_step * stride;   // row_step 2: FACR even rows
      double *u1 = u0 + (size_t)a.row_step * stride;
#pragma unroll
      for (int kk = 0; kk <= M / TT; ++kk) {
        const int n = t + kk * TT;
        if (n > M) break;
        double x = 0.0, y = 0.0;
        if (n >= 1 && n < M) {
          const double2 w = sm.xc(t, reg::sw(t), kk * TT);
          x = j0 ? w.x : 0.0;
          y = w.y;
        }
        u0[n] = x;
        u1[n] = y;
        if (last) u1[stride + n] = 0.0;
      }
    } else {
      double2 *U = static_cast<double2 *>(u);
      double2 *u0 = U + (size_t)r0 * a.row_step * stride;
#pragma unroll
      for (int kk = 0; kk <= M / TT; ++kk) {
        const int n = t + kk * TT;
        if (n > M) break;
        u0[n] = (n >= 1 && n < M && j0) ? sm.xc(t, reg::sw(t), kk * TT) : make_double2(0.0, 0.0);
        if (last) u0[stride + n] = make_double2(0.0, 0.0);
      }
    }
  }
  if constexpr (C::CL > 1) reg::seq_sync<LOGN>();
}

}  // namespace kfbi
