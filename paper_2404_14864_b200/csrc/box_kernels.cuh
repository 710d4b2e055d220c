// Box solve (Delta_h - kappa) u = rhs, dirichlet-zero closure
// (BoxSolver.solve, boxsolve.py:46-94) as three HBM passes:
//
//   rows_fwd : rhs rows (+ the sparse jump corrections of those rows,
//              interface.py:235-238 / bvp.py:319) -> DST-I along x -> panels
//   cols     : panel of columns -> DST-I along y -> / (lam_p + lam_q - kappa)
//              / (4 M^2) -> DST-I along y (adjoint engine) -> panels
//   rows_inv : panels -> DST-I along x -> u rows, exact zero ring
//
// Panel layout of the intermediate spectrum ("panels"): 32-byte column
// strips.  Real data: panel pp holds spectral x-columns 4pp..4pp+3 of every
// interior row, P[(pp*M + r)*4 + w]; complex data: 2 columns,
// P2[(pp*M + r)*2 + w].  A column pass therefore reads one contiguous
// M*32-byte slab, and a row task writes full 32-byte sectors.
//
// Real data is packed two rows (or two columns) per complex sequence.
// Global loads are batched (LB per thread in flight) before the shared-memory
// scatter so the HBM latency is overlapped.
#pragma once

#include "dst_engine.cuh"

namespace kfbi {

constexpr int LB = 8;   // global loads in flight per thread in the load phases
constexpr int DST_THREADS = 256;   // threads per DST CTA (one sequence; 3 CTAs / SM: 512 measured slower)

struct BoxArgs {
  int m, logm;
  const double2 *tw;      // packed twiddle table (twiddle_slots(m) entries)
  const double *lam;      // [m+1] (2cos(p pi/m) - 2)/h^2 at p = 1..m-1
  double kre, kim;        // kappa
  double inv4m2;          // 1 / (4 m^2), exact power of two
  void *panels;
  const int *done;        // early-exit flag (Richardson sweeps), may be null
  const double2 *twg;     // [m] exp(-2 pi i q / m)        (register engine)
  const double *sinv;     // [m] sin(pi j / m)              (register engine)
};

// Sparse right-hand-side corrections fused into the forward row pass.
template <typename T>
struct CorrArgs {
  const T *jv;            // [n_edges][3] (u, u_axis, u_axis_axis) at the crossing
  const int *row_group;   // [m+2] groups of grid row j: [row_group[j], row_group[j+1])
  const int *group_start; // [n_groups+1]
  const int *group_node;  // [n_groups] flat owner index
  const int *rec_edge;
  const double *rec_d;
  const double *rec_sigma;
};

// Correction at one irregular node: sum over its arm records, in record
// order, of sigma * (j_u + j_1 d + 0.5 j_2 d^2) (interface.py:228-237).
template <typename T>
KFBI_DEV T group_correction(const CorrArgs<T> &c, int g) {
  using S = Sc<T>;
  const int r0 = c.group_start[g], r1 = c.group_start[g + 1];
  T acc = S::zero();
  for (int r = r0; r < r1; ++r) {
    const int e = c.rec_edge[r];
    const T j0 = c.jv[3 * e], j1 = c.jv[3 * e + 1], j2 = c.jv[3 * e + 2];
    const double d = c.rec_d[r];
    T v = S::add(S::add(j0, S::rmul(j1, d)), S::rmul(S::rmul(j2, 0.5), d * d));
    v = S::rmul(v, c.rec_sigma[r]);
    acc = (r == r0) ? v : S::add(acc, v);
  }
  return acc;
}

// Dense scatter of the group sums (the standalone corrections() API).
template <typename T>
__global__ void scatter_groups_kernel(CorrArgs<T> c, int n_groups, T *out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n_groups) out[c.group_node[g]] = group_correction<T>(c, g);
}

KFBI_DEV void add_component(double2 *sm, int p, bool neg, bool imag, double v) {
  double *slot = reinterpret_cast<double *>(&sm[phys(p)]) + (imag ? 1 : 0);
  *slot += neg ? -v : v;
}
KFBI_DEV void add_corr(double2 *sm, int p, bool neg, double2 v) {
  double2 &slot = sm[phys(p)];
  slot = neg ? csub(slot, v) : cadd(slot, v);
}

// Shared-memory bytes of a kernel holding nseq sequences of length m.
inline size_t box_smem_bytes(int m, int nseq) {
  return ((size_t)nseq * m + twiddle_slots(m)) * sizeof(double2);
}

// ---------------------------------------------------------------------------
// forward row pass: one task = rows (j0, j0+1) packed (real) or row j0 (complex)
template <bool CPLX>
__global__ void __launch_bounds__(DST_THREADS)
rows_fwd_kernel(BoxArgs a, const void *__restrict__ rhs, double sign,
                CorrArgs<typename std::conditional<CPLX, double2, double>::type> corr) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  extern __shared__ double2 sm[];
  if (a.done && *a.done) return;
  const int M = a.m, logN = a.logm, tid = threadIdx.x, NT = blockDim.x;
  const int stride = M + 1;
  const int j0 = CPLX ? blockIdx.x + 1 : 2 * blockIdx.x + 1;
  const bool has2 = !CPLX && (j0 + 1 < M);
  const Twiddle tw = load_twiddles(sm + M, a.tw, M, tid, NT);

  for (int n0 = 1 + tid; n0 < M; n0 += NT * LB) {
    double2 v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int n = n0 + b * NT;
      v[b] = make_double2(0.0, 0.0);
      if (n < M && rhs != nullptr) {
        if (CPLX) {
          v[b] = static_cast<const double2 *>(rhs)[(size_t)j0 * stride + n];
        } else {
          const double *r = static_cast<const double *>(rhs);
          v[b].x = r[(size_t)j0 * stride + n];
          if (has2) v[b].y = r[(size_t)(j0 + 1) * stride + n];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int n = n0 + b * NT;
      if (n < M) {
        bool neg;
        const int p = dst_in_pos(n, logN, neg);
        const double2 x = cscale(v[b], sign);
        sm[phys(p)] = neg ? cneg(x) : x;
      }
    }
  }
  __syncthreads();
  if (corr.jv) {
    const int nrows = CPLX ? 1 : (has2 ? 2 : 1);
    for (int q = 0; q < nrows; ++q) {
      const int j = j0 + q;
      const int g0 = corr.row_group[j], g1 = corr.row_group[j + 1];
      for (int g = g0 + tid; g < g1; g += NT) {
        const T cv = group_correction<T>(corr, g);
        const int i = corr.group_node[g] - j * stride;
        bool neg;
        const int p = dst_in_pos(i, logN, neg);
        if constexpr (CPLX) add_corr(sm, p, neg, cv);
        else add_component(sm, p, neg, q == 1, cv);
      }
    }
    __syncthreads();
  }
  dst1_forward(sm, 1, logN, tw, tid, NT);

  // lane-contiguous spectral index k: conflict-free shared reads; 4 (real)
  // or 2 (complex) consecutive lanes fill one 32-byte panel sector.  The
  // padding column k = M is never written (zero since plan creation).
  const int r = j0 - 1;
  if (!CPLX) {
    double *P = static_cast<double *>(a.panels);
    for (int k = tid; k < M; k += NT) {   // k = 0 skipped: windows stay aligned
      if (k == 0) continue;
      const double2 c = sm[phys(k)];
      const int kk = k - 1;
      double *d0 = P + ((size_t)(kk >> 2) * M + r) * 4 + (kk & 3);
      d0[0] = c.x;
      d0[4] = c.y;                              // row r+1 follows row r
    }
  } else {
    double2 *P = static_cast<double2 *>(a.panels);
    for (int k = tid; k < M; k += NT) {
      if (k == 0) continue;
      const int kk = k - 1;
      P[((size_t)(kk >> 1) * M + r) * 2 + (kk & 1)] = sm[phys(k)];
    }
  }
}

// ---------------------------------------------------------------------------
// fused column pass: panel -> DST(y) -> scale -> DST(y) -> panel (in place)
// One CTA per complex sequence = half a 32-byte panel (two real columns or one
// complex column); the two halves of a panel are adjacent CTAs, so each
// 32-byte sector is read from DRAM once and served to the second CTA by L2.
template <bool CPLX>
__global__ void __launch_bounds__(DST_THREADS) cols_kernel(BoxArgs a) {
  extern __shared__ double2 sm[];
  if (a.done && *a.done) return;
  const int M = a.m, logN = a.logm, tid = threadIdx.x, NT = blockDim.x;
  const int pp = blockIdx.x >> 1, half = blockIdx.x & 1;
  double2 *P = static_cast<double2 *>(a.panels) + (size_t)pp * M * 2 + half;
  const Twiddle tw = load_twiddles(sm + M, a.tw, M, tid, NT);

  for (int r0 = tid; r0 < M - 1; r0 += NT * LB) {
    double2 v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int r = r0 + b * NT;
      if (r < M - 1) v[b] = P[2 * r];
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int r = r0 + b * NT;
      if (r < M - 1) {
        bool neg;
        const int p = phys(dst_in_pos(r + 1, logN, neg));
        sm[p] = neg ? cneg(v[b]) : v[b];
      }
    }
  }
  __syncthreads();
  dst1_forward(sm, 1, logN, tw, tid, NT);

  for (int p = tid; p < M; p += NT) {            // spectral y index (p = 0 unused)
    if (p == 0) continue;
    double2 *slot = &sm[phys(p)];
    double2 v = *slot;
    const double lp = a.lam[p];
    if (!CPLX) {
      const int kx = 4 * pp + 2 * half + 1;      // spectral x index of .x
      const double da = (lp + a.lam[kx < M ? kx : 1]) - a.kre;
      const double db = (lp + a.lam[kx + 1 < M ? kx + 1 : 1]) - a.kre;
      v.x = kx < M ? (v.x / da) * a.inv4m2 : 0.0;
      v.y = kx + 1 < M ? (v.y / db) * a.inv4m2 : 0.0;
    } else {
      const int kx = 2 * pp + half + 1;
      if (kx < M) {
        const double2 d = make_double2((lp + a.lam[kx]) - a.kre, -a.kim);
        v = cscale(cdiv(v, d), a.inv4m2);
      } else {
        v = make_double2(0.0, 0.0);
      }
    }
    *slot = v;
  }
  __syncthreads();
  dst1_adjoint(sm, 1, logN, tw, tid, NT);

  for (int r = tid; r < M - 1; r += NT) {
    bool neg;
    const double2 v = sm[phys(dst_in_pos(r + 1, logN, neg))];
    P[2 * r] = neg ? cneg(v) : v;
  }
}

// ---------------------------------------------------------------------------
// inverse row pass: panels -> DST(x) (adjoint engine, gather store) -> u rows
template <bool CPLX>
__global__ void __launch_bounds__(DST_THREADS) rows_inv_kernel(BoxArgs a, void *__restrict__ u) {
  extern __shared__ double2 sm[];
  if (a.done && *a.done) return;
  const int M = a.m, logN = a.logm, tid = threadIdx.x, NT = blockDim.x;
  const int stride = M + 1;
  const int j0 = CPLX ? blockIdx.x + 1 : 2 * blockIdx.x + 1;
  const bool has2 = !CPLX && (j0 + 1 < M);
  const int r = j0 - 1;
  const Twiddle tw = load_twiddles(sm + M, a.tw, M, tid, NT);

  for (int k0 = tid; k0 < M; k0 += NT * LB) {
    double2 v[LB];
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int k = k0 + b * NT;
      v[b] = make_double2(0.0, 0.0);
      if (k >= 1 && k < M) {
        const int kk = k - 1;
        if (!CPLX) {
          const double *s0 = static_cast<const double *>(a.panels) +
                             ((size_t)(kk >> 2) * M + r) * 4 + (kk & 3);
          v[b].x = s0[0];
          if (has2) v[b].y = s0[4];
        } else {
          v[b] = static_cast<const double2 *>(a.panels)[((size_t)(kk >> 1) * M + r) * 2 + (kk & 1)];
        }
      }
    }
#pragma unroll
    for (int b = 0; b < LB; ++b) {
      const int k = k0 + b * NT;
      if (k >= 1 && k < M) sm[phys(k)] = v[b];
    }
  }
  __syncthreads();
  dst1_adjoint(sm, 1, logN, tw, tid, NT);

  // gather + store, with the zero ring (boxsolve.py:90-93)
  if (!CPLX) {
    double *U = static_cast<double *>(u);
    double *u0 = U + (size_t)j0 * stride;
    double *u1 = U + (size_t)(j0 + 1) * stride;   // row M (ring) when !has2
    for (int n = tid; n <= M; n += NT) {
      double x = 0.0, y = 0.0;
      if (n >= 1 && n < M) {
        bool neg;
        const double2 v = sm[phys(dst_in_pos(n, logN, neg))];
        x = neg ? -v.x : v.x;
        y = neg ? -v.y : v.y;
      }
      u0[n] = x;
      u1[n] = has2 ? y : 0.0;
    }
  } else {
    double2 *U = static_cast<double2 *>(u);
    double2 *u0 = U + (size_t)j0 * stride;
    for (int n = tid; n <= M; n += NT) {
      double2 v = make_double2(0.0, 0.0);
      if (n >= 1 && n < M) {
        bool neg;
        v = sm[phys(dst_in_pos(n, logN, neg))];
        if (neg) v = cneg(v);
      }
      u0[n] = v;
    }
    if (j0 == M - 1) {
      for (int n = tid; n <= M; n += NT) U[(size_t)M * stride + n] = make_double2(0.0, 0.0);
    }
  }
  if (blockIdx.x == 0) {
    if (!CPLX) {
      double *U = static_cast<double *>(u);
      for (int n = tid; n <= M; n += NT) U[n] = 0.0;
    } else {
      double2 *U = static_cast<double2 *>(u);
      for (int n = tid; n <= M; n += NT) U[n] = make_double2(0.0, 0.0);
    }
  }
}

}  // namespace kfbi
