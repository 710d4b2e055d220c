// Per-sweep boundary kernels of the Richardson iteration:
//   jumps_d1 / jumps_d2 : compute_jumps (interface.py:171-203) with the
//                         spectral derivative of geometry.py:415-444 applied
//                         as a circulant matvec (n_ctl is any even number)
//   corr_edges          : W @ JM of corrections (interface.py:225-231), one
//                         streamed W row per unique sign-change edge (both
//                         records of an edge share theta, grid.py:243-254)
//   extract_update      : TraceExtractor.extract (bvp.py:88-104) + density
//                         update and max-norm (bvp.py:325-344), last block
//                         closes the sweep (history, convergence flag)
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace kfbi {

// Device-resident Richardson bookkeeping (one per plan).
struct RichState {
  int done;                       // 0 running, 1 converged, 2 max_iter reached
  int iters;                      // sweeps completed
  int max_iter;
  int pad0;
  double tol;
  double last_res;
  unsigned long long res_bits;    // running max |update| of the current sweep
  unsigned int arrive;            // blocks of extract_update finished
  unsigned int pad1;
};

struct CtlGeom {
  int n;                          // control points
  const double *deriv_col;        // [n] first column of d/dtheta
  const double *speed;
  const double *tangent;          // [n][2]
  const double *normal;           // [n][2]
  const double *dtan_ds;          // [n][2]
  const double *inv3;             // [n][3][3]
};

// out_i = (sum_j D[(i-j) mod n] v_j) / speed_i   (warp per output)
template <typename T>
KFBI_DEV T circ_deriv(const CtlGeom &g, const T *__restrict__ v, int i, int lane) {
  using S = Sc<T>;
  constexpr int U = 8;                // independent partial sums: U loads in flight
  T acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = S::zero();
  int j = lane;
  for (; j + 32 * (U - 1) < g.n; j += 32 * U) {
    T x[U];
    double d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int idx = i - (j + 32 * u);
      if (idx < 0) idx += g.n;
      x[u] = v[j + 32 * u];
      d[u] = __ldg(&g.deriv_col[idx]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = S::add(acc[u], S::rmul(x[u], d[u]));
  }
  for (; j < g.n; j += 32) {
    int idx = i - j;
    if (idx < 0) idx += g.n;
    acc[0] = S::add(acc[0], S::rmul(v[j], __ldg(&g.deriv_col[idx])));
  }
#pragma unroll
  for (int u = 1; u < U; ++u) acc[0] = S::add(acc[0], acc[u]);
  return acc[0];
}

// Block-wide copy global -> shared with U loads in flight per thread before
// any store (a plain strided loop waits out one L2 round trip per element).
template <int U, typename LD, typename ST>
KFBI_DEV void stage_batched(int count, LD ld, ST st) {
  const int nt = blockDim.x, tid = threadIdx.x;
  for (int base = 0; base < count; base += U * nt) {
    decltype(ld(0)) v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nt + tid;
      if (i < count) v[u] = ld(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nt + tid;
      if (i < count) st(i, v[u]);
    }
  }
}

KFBI_DEV double warp_reduce_T(double v) { return warp_sum(v); }
KFBI_DEV double2 warp_reduce_T(double2 v) {
  return make_double2(warp_sum(v.x), warp_sum(v.y));
}

// Jump system of control point i given phi_ss (the epilogue of jumps_d2).
template <typename T>
struct JumpArgs {
  const T *phi, *psi, *phi_s, *psi_s, *f_gamma;
  double fg_sign, kre, kim;
  T *jm;
};

template <typename T>
KFBI_DEV void jump_system(const CtlGeom &g, const JumpArgs<T> &a, int i, T pss) {
  using S = Sc<T>;
  const T ju = a.phi ? a.phi[i] : S::zero();
  const T ps = a.phi ? a.phi_s[i] : S::zero();
  const T pv = a.psi ? a.psi[i] : S::zero();
  const T pvs = a.psi ? a.psi_s[i] : S::zero();
  const double t1 = g.tangent[2 * i], t2 = g.tangent[2 * i + 1];
  const double dt1 = g.dtan_ds[2 * i], dt2 = g.dtan_ds[2 * i + 1];
  const T jx = S::add(S::rmul(ps, t1), S::rmul(pv, t2));
  const T jy = S::sub(S::rmul(ps, t2), S::rmul(pv, t1));
  const T r0 = S::sub(S::sub(pss, S::rmul(jx, dt1)), S::rmul(jy, dt2));
  const T r1 = S::add(S::sub(pvs, S::rmul(jx, dt2)), S::rmul(jy, dt1));
  const T r2 = S::add(S::rmul(a.f_gamma[i], a.fg_sign), S::kmul(a.kre, a.kim, ju));
  const double *A = g.inv3 + 9 * i;
  const int n = g.n;
  T *jm = a.jm;
  jm[i] = ju;
  jm[n + i] = jx;
  jm[2 * n + i] = jy;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    T v = S::add(S::add(S::rmul(r0, A[3 * r]), S::rmul(r1, A[3 * r + 1])), S::rmul(r2, A[3 * r + 2]));
    jm[(3 + r) * n + i] = v;
  }
}

// Circulant derivatives through shared memory: out_i = (sum_j D[(i-j) mod n]
// v_j) / speed_i for NV vectors (the spectral d/dtheta of geometry.py:415-426
// as its circulant column).  CTA = CIRC_OUT outputs x CIRC_CH control chunks;
// a thread keeps 4 consecutive outputs of one chunk with a sliding window of
// D (one D and NV v reads per 4 NV FMAs); the chunk partials are added in
// chunk order.  JUMPS: the jump system runs as the epilogue (jumps_d2).
constexpr int CIRC_OUT = 16, CIRC_CH = 64;
template <typename T>
inline size_t circ_smem_bytes(int n, int nv) {
  return ((size_t)((n + 1) & ~1)) * sizeof(double) + (size_t)nv * n * sizeof(T) +
         (size_t)CIRC_CH * nv * CIRC_OUT * sizeof(T);
}

template <typename T, int NV, bool JUMPS>
__global__ void __launch_bounds__(256)
circ_block_kernel(CtlGeom g, const T *__restrict__ v0, const T *__restrict__ v1, T *o0, T *o1,
                  JumpArgs<T> ja, const int *done) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char circ_sm[];
  if (done && *done) return;
  const int n = g.n, tid = threadIdx.x;
  double *Ds = reinterpret_cast<double *>(circ_sm);
  T *vs = reinterpret_cast<T *>(Ds + ((n + 1) & ~1));
  T *red = vs + NV * n;
  const bool have = v0 != nullptr;
  {
    // D and the NV vectors in the same rounds: U elements of each in flight
    // per thread (one L2 round trip per round instead of one per array)
    constexpr int U = std::is_same<T, double>::value && NV == 1 ? 12 : 6;
    const int nt = blockDim.x;
    for (int base = 0; base < n; base += U * nt) {
      double dv[U];
      T xv[NV][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * nt + tid;
        if (i < n) {
          dv[u] = g.deriv_col[i];
          if (have) {
            xv[0][u] = v0[i];
            if constexpr (NV == 2) xv[NV - 1][u] = v1[i];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * nt + tid;
        if (i < n) {
          Ds[i] = dv[u];
          if (have) {
            vs[i] = xv[0][u];
            if constexpr (NV == 2) vs[n + i] = xv[NV - 1][u];
          }
        }
      }
    }
  }
  __syncthreads();
  const int q = tid & 3, c = tid >> 2;
  const int i0 = blockIdx.x * CIRC_OUT, ib = i0 + 4 * q;
  const int j0 = (int)((long)n * c / CIRC_CH), j1 = (int)((long)n * (c + 1) / CIRC_CH);
  T acc[NV][4];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[v][r] = S::zero();
  if (have) {
    double w[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) w[r] = Ds[(((ib + r - j0) % n) + n) % n];
    for (int j = j0; j < j1; ++j) {
      const T x0 = vs[j];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[0][r] = S::add(acc[0][r], S::rmul(x0, w[r]));
      if constexpr (NV == 2) {
        const T x1 = vs[n + j];
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[1][r] = S::add(acc[1][r], S::rmul(x1, w[r]));
      }
      w[3] = w[2];
      w[2] = w[1];
      w[1] = w[0];
      int idx = ib - j - 1;
      if (idx < 0) idx += n;
      w[0] = Ds[idx];
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int r = 0; r < 4; ++r) red[(c * NV + v) * CIRC_OUT + 4 * q + r] = acc[v][r];
  __syncthreads();
  // the CIRC_CH chunk partials of an output: 8 threads sum 8 chunks each (in
  // chunk order), then a fixed shuffle tree (deterministic)
  T sum;
  {
    const int ov = tid >> 3, part = tid & 7;     // ov = v * CIRC_OUT + o
    sum = S::zero();
    if (ov < NV * CIRC_OUT) {
      const int v = ov / CIRC_OUT, o = ov - v * CIRC_OUT;
      constexpr int PER = CIRC_CH / 8;
      sum = red[((part * PER) * NV + v) * CIRC_OUT + o];
#pragma unroll
      for (int cc = 1; cc < PER; ++cc) sum = S::add(sum, red[((part * PER + cc) * NV + v) * CIRC_OUT + o]);
    }
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
      if constexpr (std::is_same<T, double>::value) sum += __shfl_down_sync(0xffffffffu, sum, off, 8);
      else {
        sum.x += __shfl_down_sync(0xffffffffu, sum.x, off, 8);
        sum.y += __shfl_down_sync(0xffffffffu, sum.y, off, 8);
      }
    }
  }
  static_assert(NV * CIRC_OUT * 8 <= 256 && CIRC_CH % 8 == 0, "circ reduction layout");
  if ((tid & 7) == 0 && (tid >> 3) < NV * CIRC_OUT) {
    const int v = (tid >> 3) / CIRC_OUT, o = (tid >> 3) - v * CIRC_OUT, i = i0 + o;
    if (i < n) {
      sum = rdiv(sum, g.speed[i]);
      if constexpr (JUMPS) {
        jump_system<T>(g, ja, i, have ? sum : S::zero());
      } else {
        (v == 0 ? o0 : o1)[i] = sum;
      }
    }
  }
}

// phi_s (and psi_s when psi != nullptr).
template <typename T>
__global__ void jumps_d1_kernel(CtlGeom g, const T *__restrict__ phi, const T *__restrict__ psi,
                                T *phi_s, T *psi_s, const int *done) {
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= g.n) return;
  const double sp = g.speed[i];
  if (phi) {
    T a = warp_reduce_T(circ_deriv<T>(g, phi, i, lane));
    if (lane == 0) phi_s[i] = rdiv(a, sp);
  }
  if (psi) {
    T b = warp_reduce_T(circ_deriv<T>(g, psi, i, lane));
    if (lane == 0) psi_s[i] = rdiv(b, sp);
  }
}

// phi_ss, then the 2x2 / 3x3 jump systems; writes JM as SoA [6][n].
template <typename T>
__global__ void jumps_d2_kernel(CtlGeom g, const T *__restrict__ phi, const T *__restrict__ psi,
                                const T *__restrict__ phi_s, const T *__restrict__ psi_s,
                                const T *__restrict__ f_gamma, double fg_sign, double kre,
                                double kim, T *jm, const int *done) {
  using S = Sc<T>;
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= g.n) return;
  T pss = S::zero();
  if (phi) pss = warp_reduce_T(circ_deriv<T>(g, phi_s, i, lane));
  if (lane != 0) return;
  const double sp = g.speed[i];
  if (phi) pss = rdiv(pss, sp);
  const T ju = phi ? phi[i] : S::zero();
  const T ps = phi ? phi_s[i] : S::zero();
  const T pv = psi ? psi[i] : S::zero();
  const T pvs = psi ? psi_s[i] : S::zero();
  const double t1 = g.tangent[2 * i], t2 = g.tangent[2 * i + 1];
  const double dt1 = g.dtan_ds[2 * i], dt2 = g.dtan_ds[2 * i + 1];
  const T jx = S::add(S::rmul(ps, t1), S::rmul(pv, t2));
  const T jy = S::sub(S::rmul(ps, t2), S::rmul(pv, t1));
  const T r0 = S::sub(S::sub(pss, S::rmul(jx, dt1)), S::rmul(jy, dt2));
  const T r1 = S::add(S::sub(pvs, S::rmul(jx, dt2)), S::rmul(jy, dt1));
  const T r2 = S::add(S::rmul(f_gamma[i], fg_sign), S::kmul(kre, kim, ju));
  const double *A = g.inv3 + 9 * i;
  const int n = g.n;
  jm[i] = ju;
  jm[n + i] = jx;
  jm[2 * n + i] = jy;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    T v = S::add(S::add(S::rmul(r0, A[3 * r]), S::rmul(r1, A[3 * r + 1])), S::rmul(r2, A[3 * r + 2]));
    jm[(3 + r) * n + i] = v;
  }
}

// ---------------------------------------------------------------------------
// Device-side setup of W (InterfaceWorkspace.__init__, interface.py:161): the
// cardinal trigonometric interpolation rows of _trig_rows (interface.py:38-52)
//   x = mod(q - theta_p + pi, 2 pi) - pi   (numpy float mod: sign of divisor)
//   D(x) = sin(m x / 2) cos(x / 2) / (m sin(x / 2)),  D = 1 where |x| < 1e-12
// element-wise with the reference's operation order; the padding column of an
// even-padded row stride is zero.  Differs from numpy only by libm rounding
// (<= a few ulp).
KFBI_DEV double np_mod(double a, double b) {
  double r = fmod(a, b);
  if (r != 0.0) {
    if ((b < 0.0) != (r < 0.0)) r += b;
  } else {
    r = copysign(0.0, b);
  }
  return r;
}

__global__ void __launch_bounds__(256)
w_build_kernel(int n_edges, int n_ctl, int ld, const double *__restrict__ edge_theta,
               const double *__restrict__ ctl_theta, double *__restrict__ W) {
  const double PI = 3.141592653589793;
  const long total = (long)n_edges * ld;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int e = (int)(i / ld), p = (int)(i - (long)e * ld);
    double v = 0.0;
    if (p < n_ctl) {
      const double x = np_mod(edge_theta[e] - ctl_theta[p] + PI, 2.0 * PI) - PI;
      const bool hit = fabs(x) < 1e-12;
      const double xs = hit ? 1.0 : x;
      const double r = sin(0.5 * n_ctl * xs) * cos(0.5 * xs) / (n_ctl * sin(0.5 * xs));
      v = hit ? 1.0 : r;
    }
    W[i] = v;
  }
}

// ---------------------------------------------------------------------------
// jv[e] = (W_e . JM_u, W_e . JM_a, W_e . JM_aa), a = x (horizontal) or y.
// A warp owns EW consecutive edges and streams their W rows once.
struct EdgeArgs {
  int n_edges, n_ctl, ld;         // ld: row stride of W (even)
  int per_warp;                   // edges per warp (<= EW of the launch)
  const double *W;
  const signed char *axis;
};

template <typename T, int EW, int U>
__global__ void __launch_bounds__(256)
corr_edges_kernel(EdgeArgs ea, const T *__restrict__ jm, T *jv, const int *done) {
  using S = Sc<T>;
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // balanced contiguous ranges of <= EW edges per warp (ea.per_warp)
  const int e0 = gw * ea.per_warp;
  const int e_end = min(e0 + ea.per_warp, ea.n_edges);
  if (e0 >= ea.n_edges) return;
  const int n = ea.n_ctl;
  const T *ju = jm, *jx = jm + n, *jy = jm + 2 * n, *jxx = jm + 3 * n, *jyy = jm + 5 * n;
  bool vert[EW];
  const double *wr[EW];
#pragma unroll
  for (int q = 0; q < EW; ++q) {
    int e = min(e0 + q, e_end - 1);
    vert[q] = ea.axis[e] != 0;
    wr[q] = ea.W + (size_t)e * ea.ld;
  }
  T acc[EW][3];
#pragma unroll
  for (int q = 0; q < EW; ++q) acc[q][0] = acc[q][1] = acc[q][2] = S::zero();
  // 16-byte W loads (rows padded to an even length with zeros), two pairs of
  // control points per lane per iteration: 2*EW streaming loads in flight
  // U iterations of EW rows are loaded before any is used: U*EW 16-byte
  // streaming loads in flight per lane (the compiler does not hoist them
  // across the FMA chains on its own).
  const int n2 = ea.ld >> 1;
  for (int i0 = lane; i0 < n2; i0 += 32 * U) {
    double2 w2[U][EW];
    // one asm statement per 4 rows: the loads issue back to back, ahead of
    // any use (ptxas otherwise interleaves them with the FMA chains)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i2 = i0 + 32 * u;
      const int ii = i2 < n2 ? i2 : 0;
#pragma unroll
      for (int q0 = 0; q0 < EW; q0 += 4) {
        const double2 *a0 = reinterpret_cast<const double2 *>(wr[q0]) + ii;
        const double2 *a1 = reinterpret_cast<const double2 *>(wr[q0 + 1]) + ii;
        const double2 *a2 = reinterpret_cast<const double2 *>(wr[q0 + 2]) + ii;
        const double2 *a3 = reinterpret_cast<const double2 *>(wr[q0 + 3]) + ii;
        asm volatile(
            "ld.global.cs.v2.f64 {%0,%1}, [%8];\n\t"
            "ld.global.cs.v2.f64 {%2,%3}, [%9];\n\t"
            "ld.global.cs.v2.f64 {%4,%5}, [%10];\n\t"
            "ld.global.cs.v2.f64 {%6,%7}, [%11];"
            : "=d"(w2[u][q0].x), "=d"(w2[u][q0].y), "=d"(w2[u][q0 + 1].x), "=d"(w2[u][q0 + 1].y),
              "=d"(w2[u][q0 + 2].x), "=d"(w2[u][q0 + 2].y), "=d"(w2[u][q0 + 3].x),
              "=d"(w2[u][q0 + 3].y)
            : "l"(a0), "l"(a1), "l"(a2), "l"(a3));
      }
      if (i2 >= n2)
#pragma unroll
        for (int q = 0; q < EW; ++q) w2[u][q] = make_double2(0.0, 0.0);
    }

#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = min(2 * (i0 + 32 * u) + h, n - 1);
        const T a0 = ju[i], ax = jx[i], ay = jy[i], axx = jxx[i], ayy = jyy[i];
#pragma unroll
        for (int q = 0; q < EW; ++q) {
          const double w = h ? w2[u][q].y : w2[u][q].x;
          acc[q][0] = S::add(acc[q][0], S::rmul(a0, w));
          acc[q][1] = S::add(acc[q][1], S::rmul(vert[q] ? ay : ax, w));
          acc[q][2] = S::add(acc[q][2], S::rmul(vert[q] ? ayy : axx, w));
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < EW; ++q) {
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[q][c] = warp_reduce_T(acc[q][c]);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < EW; ++q) {
      if (e0 + q < e_end) {
        jv[3 * (e0 + q)] = acc[q][0];
        jv[3 * (e0 + q) + 1] = acc[q][1];
        jv[3 * (e0 + q) + 2] = acc[q][2];
      }
    }
  }
}

// Same product with the jump matrix staged in shared memory: a CTA of
// CE_WARPS warps owns a contiguous block of edges and walks the controls in
// chunks of CE_CK; each chunk of the five used JM columns is read from L2
// ONCE per CTA (the per-warp form above re-reads all of JM per warp: 16x the W
// bytes of L2 traffic at star3 c128) and kept de-interleaved by parity so the
// lanes' pair reads are conflict free.  The chunk's W loads are issued before
// the staging, so HBM latency overlaps it.
constexpr int CE_WARPS = 16;

template <typename T, int EW>
__global__ void __launch_bounds__(CE_WARPS * 32, 1)
corr_edges_smem_kernel(EdgeArgs ea, const T *__restrict__ jm, T *jv, const int *done) {
  using S = Sc<T>;
  // control pairs per lane per chunk: UP * EW 16-byte W loads in flight per
  // lane within the 128-register budget of 16 warps per SM
  constexpr int UP = sizeof(T) == 16 && EW >= 4 ? 2 : 4;
  constexpr int CE_CK = 64 * UP;
  __shared__ T js[5][2][CE_CK / 2];
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * CE_WARPS + (threadIdx.x >> 5);
  const int e0 = gw * ea.per_warp;
  const int e_end = min(e0 + ea.per_warp, ea.n_edges);
  const int nq = e_end - e0;                     // edges of this warp (<= 0: staging only)
  const int n = ea.n_ctl;
  bool vert[EW];
  const double2 *wr[EW];
#pragma unroll
  for (int q = 0; q < EW; ++q) {
    const int e = nq > 0 ? e0 + min(q, nq - 1) : 0;
    vert[q] = ea.axis[e] != 0;
    wr[q] = reinterpret_cast<const double2 *>(ea.W + (size_t)e * ea.ld);
  }
  T acc[EW][3];
#pragma unroll
  for (int q = 0; q < EW; ++q) acc[q][0] = acc[q][1] = acc[q][2] = S::zero();
  const int n2 = ea.ld >> 1;
  for (int c0 = 0; c0 < n; c0 += CE_CK) {
    double2 w2[UP][EW];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int i2 = (c0 >> 1) + lane + 32 * u;
      const bool ok = i2 < n2;
#pragma unroll
      for (int q = 0; q < EW; ++q) {
        if (ok && q < nq) {
          asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];"
                       : "=d"(w2[u][q].x), "=d"(w2[u][q].y) : "l"(wr[q] + i2));
        } else {
          w2[u][q] = make_double2(0.0, 0.0);
        }
      }
    }
    __syncthreads();                             // the previous chunk's reads are done
    for (int idx = threadIdx.x; idx < 5 * CE_CK; idx += CE_WARPS * 32) {
      const int col = idx / CE_CK, k = idx - col * CE_CK, i = c0 + k;
      const int off = col == 4 ? 5 : col;        // u, u_x, u_y, u_xx, u_yy
      js[col][k & 1][k >> 1] = i < n ? jm[(size_t)off * n + i] : S::zero();
    }
    __syncthreads();
    if (nq > 0) {
#pragma unroll
      for (int u = 0; u < UP; ++u) {
        const int k2 = lane + 32 * u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const T a0 = js[0][h][k2], ax = js[1][h][k2], ay = js[2][h][k2], axx = js[3][h][k2],
                  ayy = js[4][h][k2];
#pragma unroll
          for (int q = 0; q < EW; ++q) {
            const double w = h ? w2[u][q].y : w2[u][q].x;
            acc[q][0] = S::add(acc[q][0], S::rmul(a0, w));
            acc[q][1] = S::add(acc[q][1], S::rmul(vert[q] ? ay : ax, w));
            acc[q][2] = S::add(acc[q][2], S::rmul(vert[q] ? ayy : axx, w));
          }
        }
      }
    }
  }
  if (nq <= 0) return;
#pragma unroll
  for (int q = 0; q < EW; ++q) {
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[q][c] = warp_reduce_T(acc[q][c]);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < EW; ++q) {
      if (q < nq) {
        jv[3 * (e0 + q)] = acc[q][0];
        jv[3 * (e0 + q) + 1] = acc[q][1];
        jv[3 * (e0 + q) + 2] = acc[q][2];
      }
    }
  }
}

// The same with ALL of the five used JM columns staged once per CTA (when
// they fit in shared memory: n_ctl <= ~2,800 complex / ~5,600 real): no
// barrier inside the control loop, so the warps drift apart and one warp's
// W loads overlap another's FMAs.
template <typename T, int EW>
__global__ void __launch_bounds__(CE_WARPS * 32, 1)
corr_edges_full_kernel(EdgeArgs ea, const T *__restrict__ jm, T *jv, const int *done) {
  using S = Sc<T>;
  constexpr int UP = sizeof(T) == 16 && EW >= 4 ? 2 : 4;
  extern __shared__ __align__(16) unsigned char ce_smem[];
  if (done && *done) return;
  const int n = ea.n_ctl;
  const int nh = (n + 1) >> 1;                   // pairs per parity
  T *js = reinterpret_cast<T *>(ce_smem);        // [5][2][nh]
  for (int idx = threadIdx.x; idx < 5 * 2 * nh; idx += CE_WARPS * 32) {
    const int col = idx / (2 * nh), r = idx - col * 2 * nh, h = r / nh, k2 = r - h * nh;
    const int i = 2 * k2 + h;
    const int off = col == 4 ? 5 : col;          // u, u_x, u_y, u_xx, u_yy
    js[idx] = i < n ? jm[(size_t)off * n + i] : S::zero();
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * CE_WARPS + (threadIdx.x >> 5);
  const int e0 = gw * ea.per_warp;
  const int e_end = min(e0 + ea.per_warp, ea.n_edges);
  const int nq = e_end - e0;
  if (nq <= 0) return;
  bool vert[EW];
  const double2 *wr[EW];
#pragma unroll
  for (int q = 0; q < EW; ++q) {
    const int e = e0 + min(q, nq - 1);
    vert[q] = ea.axis[e] != 0;
    wr[q] = reinterpret_cast<const double2 *>(ea.W + (size_t)e * ea.ld);
  }
  T acc[EW][3];
#pragma unroll
  for (int q = 0; q < EW; ++q) acc[q][0] = acc[q][1] = acc[q][2] = S::zero();
  const int n2 = ea.ld >> 1;
  auto J = [&](int col, int h, int k2) -> T { return js[(col * 2 + h) * nh + k2]; };
  for (int c2 = 0; c2 < n2; c2 += 32 * UP) {     // control pairs c2 + lane + 32 u
    double2 w2[UP][EW];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int i2 = c2 + lane + 32 * u;
      const bool ok = i2 < n2;
#pragma unroll
      for (int q = 0; q < EW; ++q) {
        if (ok && q < nq) {
          asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];"
                       : "=d"(w2[u][q].x), "=d"(w2[u][q].y) : "l"(wr[q] + i2));
        } else {
          w2[u][q] = make_double2(0.0, 0.0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int k2 = min(c2 + lane + 32 * u, nh - 1);   // pairs past n: W is zero there
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const T a0 = J(0, h, k2), ax = J(1, h, k2), ay = J(2, h, k2), axx = J(3, h, k2),
                ayy = J(4, h, k2);
#pragma unroll
        for (int q = 0; q < EW; ++q) {
          const double w = h ? w2[u][q].y : w2[u][q].x;
          acc[q][0] = S::add(acc[q][0], S::rmul(a0, w));
          acc[q][1] = S::add(acc[q][1], S::rmul(vert[q] ? ay : ax, w));
          acc[q][2] = S::add(acc[q][2], S::rmul(vert[q] ? ayy : axx, w));
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < EW; ++q) {
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[q][c] = warp_reduce_T(acc[q][c]);
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < EW; ++q) {
      if (q < nq) {
        jv[3 * (e0 + q)] = acc[q][0];
        jv[3 * (e0 + q) + 1] = acc[q][1];
        jv[3 * (e0 + q) + 2] = acc[q][2];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Matrix-free edge values (the trig branch of interp_rows, interface.py:38-52,
// 70-75).  For the reference's equispaced controls theta_j = 2 pi j / n (n
// even) the cardinal kernel D(x) = sin(n x/2) cos(x/2) / (n sin(x/2)) is the
// trigonometric interpolant 1/n [1 + 2 sum_{k=1}^{n/2-1} cos(k x) + cos(n x/2)],
// so with F_k = sum_j f_j e^{-2 pi i j k / n} (the DFT of a real column f)
//   (W f)(theta) = 1/n [F_0 + 2 sum_{k=1}^{n/2-1} Re(e^{i k theta} F_k)
//                       + cos(n theta / 2) F_{n/2}].
// Two kernels replace the n_edges x n_ctl W stream (680 MB at 4096^2 flower in
// the reference, 5.4 GB at 16384^2): the spectrum of the five used JM columns
// (u, ux, uy, uxx, uyy; real and imaginary parts separately for c128) by a
// direct DFT, then one sum over k per edge.  The exact angles k theta come
// from an exact product (fma) and a first-order correction of sincos, the
// in-between powers from one rotation per 32 k; deviation from W . JM is the
// conditioning of the reference formula itself (k ulp(theta), <= 1e-12).
constexpr int SPEC_COLS = 5;                     // JM columns u, ux, uy, uxx, uyy
KFBI_DEV int spec_jm_col(int c) { return c < 4 ? c : 5; }

// e^{i a b} for a large product a b: exact product p + e, sincos(p) corrected
KFBI_DEV double2 cis_product(double a, double b) {
  const double p = a * b;
  const double e = fma(a, b, -p);
  double sp, cp;
  sincos(p, &sp, &cp);
  return make_double2(fma(-e, sp, cp), fma(e, cp, sp));
}

// Spectrum F_k (k < K = n/2 + 1) of the used JM columns.  CTA (x, y): lane =
// frequency k = 32 x + lane, warp w and split y cover the control range
// [(y W + w) n / (W Y), ...).  e^{-2 pi i j k / n} is exact from the index
// (j k mod n) every 32 controls and advanced by one rotation in between.  The
// W partial sums of a CTA are added in warp order in shared memory, the Y
// CTA partials of a frequency block by the last CTA to finish it, in split
// order (deterministic; the block counter resets itself).
__host__ __device__ __forceinline__ int jn_max(int n, int Y) { return (n + Y - 1) / Y + 1; }

template <typename T>
__global__ void __launch_bounds__(512)
spec_block_kernel(int n, int K, const T *__restrict__ jm, double2 *__restrict__ part,
                  double2 *__restrict__ spec, unsigned int *counters, int clustered) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
  constexpr int R = SPEC_COLS * NP;
  extern __shared__ double2 red_sm[];                   // [W][R][32], then the staged columns
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Y = gridDim.y, y = blockIdx.y;
  auto red = [&](int x, int r) -> double2 & { return red_sm[((size_t)x * R + r) * 32 + lane]; };
  const int k = blockIdx.x * 32 + lane;
  // the CTA's control range, staged column-major [SPEC_COLS][jn] in shared memory
  const int cj0 = (int)((long)n * y / Y), cj1 = (int)((long)n * (y + 1) / Y), jn = cj1 - cj0;
  T *fs = reinterpret_cast<T *>(red_sm + (size_t)nw * R * 32);
  double2 *fs_end = reinterpret_cast<double2 *>(
      reinterpret_cast<unsigned char *>(fs) + (((size_t)SPEC_COLS * (jn_max(n, Y)) * sizeof(T) + 15) & ~(size_t)15));
  stage_batched<8>(SPEC_COLS * jn, [&](int i) {
    const int c = i / jn, j = i - c * jn;
    return jm[(size_t)spec_jm_col(c) * n + cj0 + j];
  }, [&](int i, T x) { fs[i] = x; });
  __syncthreads();
  const int j0 = cj0 + (int)((long)jn * w / nw), j1 = cj0 + (int)((long)jn * (w + 1) / nw);
  double2 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = make_double2(0.0, 0.0);
  if (k < K) {
    double ss, cs;
    sincospi(-2.0 * (double)k / n, &ss, &cs);
    const double2 step = make_double2(cs, ss);
    double2 wk = make_double2(1.0, 0.0);
    int idx = (int)(((long)j0 * k) % n);                 // j k mod n, advanced by k per control
    for (int j = j0; j < j1; ++j) {
      if (((j - j0) & 31) == 0) {
        double sw, cw;
        sincospi(-2.0 * (double)idx / n, &sw, &cw);
        wk = make_double2(cw, sw);
      }
#pragma unroll
      for (int c = 0; c < SPEC_COLS; ++c) {
        const T v = fs[c * jn + (j - cj0)];
        if constexpr (NP == 1) {
          acc[c].x = fma(v, wk.x, acc[c].x);
          acc[c].y = fma(v, wk.y, acc[c].y);
        } else {
          acc[c].x = fma(v.x, wk.x, acc[c].x);
          acc[c].y = fma(v.x, wk.y, acc[c].y);
          acc[SPEC_COLS + c].x = fma(v.y, wk.x, acc[SPEC_COLS + c].x);
          acc[SPEC_COLS + c].y = fma(v.y, wk.y, acc[SPEC_COLS + c].y);
        }
      }
      wk = cmul(wk, step);
      idx += k;
      if (idx >= n) idx -= n;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) red(w, r) = acc[r];
  __syncthreads();
  if (clustered) {
    // the Y splits of a frequency block form one thread-block cluster: the
    // CTA column sums meet in the rank-0 CTA's view of distributed shared
    // memory, added in split order (the order of the global-partials path)
    double2 *csum = fs_end;                          // [R][32] after the staged columns
    for (int r = w; r < R; r += nw) {
      double2 sum = red(0, r);
      for (int x = 1; x < nw; ++x) sum = cadd(sum, red(x, r));
      csum[r * 32 + lane] = sum;
    }
    auto cl = cooperative_groups::this_cluster();
    cl.sync();
    if (cl.block_rank() == 0 && k < K)
      for (int r = w; r < R; r += nw) {
        double2 sum = csum[r * 32 + lane];
        for (int x = 1; x < Y; ++x) sum = cadd(sum, cl.map_shared_rank(csum, x)[r * 32 + lane]);
        spec[(size_t)r * K + k] = sum;
      }
    cl.sync();                                       // peers' shared memory read
    return;
  }
  // column r's warp partials summed by warp r (warp order: deterministic)
  if (k < K)
    for (int r = w; r < R; r += nw) {
      double2 sum = red(0, r);
      for (int x = 1; x < nw; ++x) sum = cadd(sum, red(x, r));
      if (Y == 1) spec[(size_t)r * K + k] = sum;
      else part[((size_t)y * R + r) * K + k] = sum;
    }
  if (Y == 1) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[blockIdx.x], 1u) == (unsigned)(Y - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (k < K)
    for (int r = w; r < R; r += nw) {
      double2 sum = __ldcg(&part[(size_t)r * K + k]);
      for (int x = 1; x < Y; ++x) sum = cadd(sum, __ldcg(&part[((size_t)x * R + r) * K + k]));
      spec[(size_t)r * K + k] = sum;
    }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

// One group of EB edges of one axis (the host orders the edges by axis and
// pads each class to whole groups; perm = -1 marks a pad): lane l sums
// k = 1 + l + 32 i (k < n/2) over the three columns (u, u_a, u_aa) of the
// group's axis.  F(col, k) returns the spectrum entry.
template <typename T, int EB, typename FN>
KFBI_DEV void edge_group(int g, int n, int K, const int *__restrict__ perm, const double *__restrict__ theta,
                         const signed char *__restrict__ axis, int kbeg, int kend, double (&acc)[EB][6],
                         double2 (&z)[EB], const double2 (&z32)[EB], int ca, FN F) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
  for (int k = kbeg; k < kend; k += 32) {
    double2 f[NP][3];
#pragma unroll
    for (int h = 0; h < NP; ++h) {
      f[h][0] = F(h * SPEC_COLS, k);
      f[h][1] = F(h * SPEC_COLS + ca, k);
      f[h][2] = F(h * SPEC_COLS + ca + 2, k);
    }
#pragma unroll
    for (int q = 0; q < EB; ++q) {
#pragma unroll
      for (int h = 0; h < NP; ++h)
#pragma unroll
        for (int c = 0; c < 3; ++c)     // Re(z F) = z.x F.x - z.y F.y
          acc[q][3 * h + c] = fma(z[q].x, f[h][c].x, fma(-z[q].y, f[h][c].y, acc[q][3 * h + c]));
      z[q] = cmul(z[q], z32[q]);
    }
  }
}

template <typename T, int EB>
KFBI_DEV void edge_group_begin(int g, const int *__restrict__ perm, const double *__restrict__ theta,
                               const signed char *__restrict__ axis, int lane, int (&eid)[EB],
                               double (&th)[EB], double2 (&z)[EB], double2 (&z32)[EB], int &ca,
                               double (&acc)[EB][6]) {
  ca = 1;
#pragma unroll
  for (int q = EB - 1; q >= 0; --q) {
    eid[q] = perm[g * EB + q];
    const int e = eid[q] >= 0 ? eid[q] : 0;
    th[q] = theta[e];
    if (eid[q] >= 0) ca = axis[e] != 0 ? 2 : 1;   // uniform over the group's real edges
    z[q] = cis_product((double)(1 + lane), th[q]);
    z32[q] = cis_product(32.0, th[q]);
#pragma unroll
    for (int c = 0; c < 6; ++c) acc[q][c] = 0.0;
  }
}

template <typename T, int EB, typename FN>
KFBI_DEV void edge_group_end(int n, int lane, const int (&eid)[EB], const double (&th)[EB], int ca,
                             double (&acc)[EB][6], T *jv, FN F) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
#pragma unroll
  for (int q = 0; q < EB; ++q)
#pragma unroll
    for (int c = 0; c < 3 * NP; ++c) acc[q][c] = warp_sum(acc[q][c]);
  if (lane >= EB) return;
  double out[6];
  double tq = th[0];
  int e = eid[0];
#pragma unroll
  for (int c = 0; c < 6; ++c) out[c] = acc[0][c];
#pragma unroll
  for (int q = 1; q < EB; ++q)
    if (lane == q) {
#pragma unroll
      for (int c = 0; c < 6; ++c) out[c] = acc[q][c];
      tq = th[q];
      e = eid[q];
    }
  if (e < 0) return;
  const double cn = cis_product(0.5 * n, tq).x;         // cos(n theta / 2)
  const double inv_n = 1.0 / n;
  const int cols[3] = {0, ca, ca + 2};
  double res[6];
#pragma unroll
  for (int h = 0; h < NP; ++h)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      res[3 * h + c] = (F(h * SPEC_COLS + cols[c], 0).x + 2.0 * out[3 * h + c] +
                        cn * F(h * SPEC_COLS + cols[c], n / 2).x) * inv_n;
  T *o = jv + 3 * (size_t)e;
  if constexpr (NP == 1) {
    o[0] = res[0];
    o[1] = res[1];
    o[2] = res[2];
  } else {
    o[0] = make_double2(res[0], res[3]);
    o[1] = make_double2(res[1], res[4]);
    o[2] = make_double2(res[2], res[5]);
  }
}

// Spectrum resident in shared memory (R K 16 bytes fit): one CTA per SM
// loads it once; its warps walk the edge groups.
template <typename T, int EB>
__global__ void __launch_bounds__(512, 1)
edges_spectral_res_kernel(int ngroups, int n, int K, const int *__restrict__ perm,
                          const double *__restrict__ theta, const signed char *__restrict__ axis,
                          const double2 *__restrict__ spec, T *jv, const int *done) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
  constexpr int R = SPEC_COLS * NP;
  extern __shared__ double2 fsm[];                       // [R][K]
  if (done && *done) return;
  stage_batched<16>(R * K, [&](int i) { return spec[i]; }, [&](int i, double2 x) { fsm[i] = x; });
  __syncthreads();
  const int lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  auto F = [&](int r, int k) { return fsm[(size_t)r * K + k]; };
  for (int g = blockIdx.x * nwarps + (threadIdx.x >> 5); g < ngroups; g += gridDim.x * nwarps) {
    int eid[EB], ca;
    double th[EB], acc[EB][6];
    double2 z[EB], z32[EB];
    edge_group_begin<T, EB>(g, perm, theta, axis, lane, eid, th, z, z32, ca, acc);
    edge_group<T, EB>(g, n, K, perm, theta, axis, 1 + lane, n / 2, acc, z, z32, ca, F);
    edge_group_end<T, EB>(n, lane, eid, th, ca, acc, jv, F);
  }
}

// Large n (C5): one group per warp, the spectrum staged in chunks of
// SPEC_KC frequencies shared by the CTA's warps.
constexpr int SPEC_KC = 512;
template <typename T, int EB>
__global__ void __launch_bounds__(256)
edges_spectral_kernel(int ngroups, int n, int K, const int *__restrict__ perm,
                      const double *__restrict__ theta, const signed char *__restrict__ axis,
                      const double2 *__restrict__ spec, T *jv, const int *done) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
  constexpr int R = SPEC_COLS * NP;
  extern __shared__ double2 fsm[];                       // [R][SPEC_KC]
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = g < ngroups;
  int eid[EB], ca = 1;
  double th[EB], acc[EB][6];
  double2 z[EB], z32[EB];
  if (active) edge_group_begin<T, EB>(g, perm, theta, axis, lane, eid, th, z, z32, ca, acc);
  const int kmax = n / 2;
  for (int kc0 = 1; kc0 < kmax; kc0 += SPEC_KC) {
    const int kn = min(SPEC_KC, kmax - kc0);
    __syncthreads();
    for (int i = threadIdx.x; i < R * kn; i += blockDim.x) {
      const int r = i / kn, kk = i - r * kn;
      fsm[r * SPEC_KC + kk] = spec[(size_t)r * K + kc0 + kk];
    }
    __syncthreads();
    auto F = [&](int r, int k) { return fsm[r * SPEC_KC + (k - kc0)]; };
    if (active) edge_group<T, EB>(g, n, K, perm, theta, axis, kc0 + lane, kc0 + kn, acc, z, z32, ca, F);
  }
  if (!active) return;
  auto FG = [&](int r, int k) { return spec[(size_t)r * K + k]; };
  edge_group_end<T, EB>(n, lane, eid, th, ca, acc, jv, FG);
}

// ---------------------------------------------------------------------------
struct ExtractArgs {
  int n, m;
  double h, inv_h;
  const int *stencil;             // [n][6]
  const double *ainv_rows;        // [n][3][6]
  const double *jcoef;            // [n][6][6]
  const double *normal;           // [n][2]
  // OneSidedExtractor (bvp.py:115-228), Neumann BVPs; null -> six-point
  const int *os_stencil;          // [n][7] interior nodes
  const double *os_rows;          // [n][3][7] rows 0..2 of inv(A)
  const unsigned char *os_fb;     // [n] 1: fall back to the six-point stencil
};

// (u+, ux+, uy+) at control point p (bvp.py:98-104) from the six stencil
// values u6(s) of the straddling stencil.
template <typename T, typename U6>
KFBI_DEV void extract_point_v(const ExtractArgs &x, U6 u6, const T *__restrict__ jm, int p, T &tu,
                              T &tx, T &ty) {
  using S = Sc<T>;
  T jp[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) jp[k] = jm[k * x.n + p];
  T vals[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const double *jc = x.jcoef + 36 * p + 6 * s;
    T corr = S::rmul(jp[0], jc[0]);
#pragma unroll
    for (int k = 1; k < 6; ++k) corr = S::add(corr, S::rmul(jp[k], jc[k]));
    vals[s] = S::add(u6(s), corr);
  }
  T c[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const double *ar = x.ainv_rows + 18 * p + 6 * r;
    T acc = S::rmul(vals[0], ar[0]);
#pragma unroll
    for (int s = 1; s < 6; ++s) acc = S::add(acc, S::rmul(vals[s], ar[s]));
    c[r] = acc;
  }
  tu = c[0];
  tx = rdiv(c[1], x.h);
  ty = rdiv(c[2], x.h);
}

template <typename T>
KFBI_DEV void extract_point(const ExtractArgs &x, const T *__restrict__ u, const T *__restrict__ jm,
                            int p, T &tu, T &tx, T &ty) {
  extract_point_v<T>(x, [&](int s) { return u[x.stencil[6 * p + s]]; }, jm, p, tu, tx, ty);
}

// The extractor of the BVP kind: one-sided rows . u[7 nodes] (bvp.py:215-221)
// with the straddling fallback (bvp.py:222-227: the fallback's gradient goes
// through * h / h like the reference's coefficient array), or the six-point
// straddling stencil.  u6(s) / u7(k): field values at the stencil nodes.
template <typename T, typename U6, typename U7>
KFBI_DEV void extract_any_v(const ExtractArgs &x, U6 u6, U7 u7, const T *__restrict__ jm, int p,
                            T &tu, T &tx, T &ty) {
  using S = Sc<T>;
  if (x.os_stencil && !x.os_fb[p]) {
    T v[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) v[k] = u7(k);
    T c[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const double *rr = x.os_rows + 21 * p + 7 * r;
      T acc = S::rmul(v[0], rr[0]);
#pragma unroll
      for (int k = 1; k < 7; ++k) acc = S::add(acc, S::rmul(v[k], rr[k]));
      c[r] = acc;
    }
    tu = c[0];
    tx = rdiv(c[1], x.h);
    ty = rdiv(c[2], x.h);
    return;
  }
  extract_point_v<T>(x, u6, jm, p, tu, tx, ty);
  if (x.os_stencil) {
    tx = rdiv(S::rmul(tx, x.h), x.h);
    ty = rdiv(S::rmul(ty, x.h), x.h);
  }
}

template <typename T>
KFBI_DEV void extract_any(const ExtractArgs &x, const T *__restrict__ u, const T *__restrict__ jm,
                          int p, T &tu, T &tx, T &ty) {
  extract_any_v<T>(
      x, [&](int s) { return u[x.stencil[6 * p + s]]; },
      [&](int k) { return u[x.os_stencil[7 * p + k]]; }, jm, p, tu, tx, ty);
}

// ---- slab-decomposed sweep (dist.py): stencil values of one row slab ----
// vals[13 p + s] (six-point, s < 6) and vals[13 p + 6 + k] (one-sided) =
// u at the node when its grid row lies in [row0, row0 + rows), else 0; the
// sum over the ranks' buffers (all-reduce) is the full stencil data.
constexpr int SLAB_VALS = 13;

template <typename T>
__global__ void __launch_bounds__(256)
slab_stencil_kernel(ExtractArgs x, int row0, int rows, const T *__restrict__ u_slab, T *vals) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= x.n) return;
  const int stride = x.m + 1;
  auto pick = [&](int node) -> T {
    const int j = node / stride;
    if (j < row0 || j >= row0 + rows) return Sc<T>::zero();
    return u_slab[(size_t)(j - row0) * stride + (node - j * stride)];
  };
#pragma unroll
  for (int s = 0; s < 6; ++s) vals[SLAB_VALS * p + s] = pick(x.stencil[6 * p + s]);
#pragma unroll
  for (int k = 0; k < 7; ++k)
    vals[SLAB_VALS * p + 6 + k] = x.os_stencil ? pick(x.os_stencil[7 * p + k]) : Sc<T>::zero();
}

// Extraction from reduced stencil values + density update + residual; the
// last block closes the sweep (same arithmetic as extract_update_kernel).
template <typename T>
__global__ void __launch_bounds__(256)
extract_update_vals_kernel(ExtractArgs x, const T *__restrict__ vals, const T *__restrict__ jm,
                           const T *__restrict__ g, T *density, T *trace_u, T *trace_un,
                           double gamma, int dirichlet, RichState *st, double *history);

template <typename T>
__global__ void __launch_bounds__(256)
extract_kernel(ExtractArgs x, const T *__restrict__ u, const T *__restrict__ jm, T *out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= x.n) return;
  T tu, tx, ty;
  extract_any<T>(x, u, jm, p, tu, tx, ty);
  out[p] = tu;
  out[x.n + p] = tx;
  out[2 * x.n + p] = ty;
}

// Closes a sweep: max-norm into the state, last block decides (bvp.py:333-344).
KFBI_DEV void sweep_close(double mag, RichState *st, double *history) {
  __shared__ double red[32];
  __shared__ bool is_last;
  mag = warp_nanmax(mag);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = mag;
  __syncthreads();
  if (wid == 0) {
    double v = lane < (blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_nanmax(v);
    if (lane == 0) {
      atomic_max_nonneg(&st->res_bits, v);
      __threadfence();
      unsigned int ticket = atomicAdd(&st->arrive, 1u);
      is_last = ticket == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    unsigned long long bits = atomicAdd(&st->res_bits, 0ull);
    double res = __longlong_as_double((long long)bits);
    int it = st->iters + 1;
    history[it - 1] = res;
    st->iters = it;
    st->last_res = res;
    if (res <= st->tol) st->done = 1;
    else if (it >= st->max_iter) st->done = 2;
    st->res_bits = 0ull;
    st->arrive = 0u;
  }
}

// Extraction + density update + residual; the last block closes the sweep.
template <typename T>
__global__ void __launch_bounds__(256)
extract_update_kernel(ExtractArgs x, const T *__restrict__ u, const T *__restrict__ jm,
                      const T *__restrict__ g, T *density, T *trace_u, T *trace_un,
                      double gamma, int dirichlet, RichState *st, double *history) {
  using S = Sc<T>;
  if (st->done) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double mag = 0.0;
  if (p < x.n) {
    T tu, tx, ty;
    extract_any<T>(x, u, jm, p, tu, tx, ty);
    const double nx = x.normal[2 * p], ny = x.normal[2 * p + 1];
    T tun = S::add(S::rmul(tx, nx), S::rmul(ty, ny));
    T target = dirichlet ? tu : tun;
    T upd = S::rmul(S::sub(g[p], target), gamma);
    density[p] = S::add(density[p], upd);
    trace_u[p] = tu;
    trace_un[p] = tun;
    mag = S::abs(upd);
  }
  sweep_close(mag, st, history);
}

template <typename T>
__global__ void __launch_bounds__(256)
extract_update_vals_kernel(ExtractArgs x, const T *__restrict__ vals, const T *__restrict__ jm,
                           const T *__restrict__ g, T *density, T *trace_u, T *trace_un,
                           double gamma, int dirichlet, RichState *st, double *history) {
  using S = Sc<T>;
  if (st->done) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double mag = 0.0;
  if (p < x.n) {
    T tu, tx, ty;
    extract_any_v<T>(
        x, [&](int s) { return vals[SLAB_VALS * p + s]; },
        [&](int k) { return vals[SLAB_VALS * p + 6 + k]; }, jm, p, tu, tx, ty);
    const double nx = x.normal[2 * p], ny = x.normal[2 * p + 1];
    T tun = S::add(S::rmul(tx, nx), S::rmul(ty, ny));
    T target = dirichlet ? tu : tun;
    T upd = S::rmul(S::sub(g[p], target), gamma);
    density[p] = S::add(density[p], upd);
    trace_u[p] = tu;
    trace_un[p] = tun;
    mag = S::abs(upd);
  }
  sweep_close(mag, st, history);
}

// ---------------------------------------------------------------------------
// Operator form of the Richardson sweep.
//
// The sweep map phi -> trace(phi) is affine with a linear part T fixed by the
// geometry and kappa (jumps -> corrections -> box solve -> extraction,
// bvp.py:313-323).  The plan can hold T explicitly (column p = the pipeline
// applied to the unit density e_p with F = 0, f_gamma = 0).  Sweep 1 of a
// solve always runs the full pipeline; sweeps k >= 2 then evaluate
//     trace_k = trace_1 + T (phi_k - phi_0)
// which is the same affine map (identical iterates up to rounding), and the
// converging sweep's field is recomputed by the full pipeline from the
// density before its update.

template <typename T>
__global__ void unit_vector_kernel(T *v, int n, int p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] = (i == p) ? Sc<T>::one() : Sc<T>::zero();
}

// Column p of the trace operator, stored column-major: Tcm[p * n + q] = the
// target trace of an extraction out[3][n] = (u+, ux+, uy+): u+ (Dirichlet) or
// d_n u+ = ux+ nx + uy+ ny (Neumann).
template <typename T>
__global__ void op_column_kernel(int n, int p, const T *out, const double *normal, int neumann,
                                 T *Tcm) {
  using S = Sc<T>;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  Tcm[(size_t)p * n + q] =
      neumann ? S::add(S::rmul(out[n + q], normal[2 * q]), S::rmul(out[2 * n + q], normal[2 * q + 1]))
              : out[q];
}

// All operator sweeps of one solve in ONE cooperative launch, with the trace
// operator held on chip across the sweeps (bvp.py:312-344 semantics).
//
// CTA c owns rows [c R, c R + R) of T (one CTA per SM); lane = row within a
// 32-row tile, warp w = columns w, w + NW, ...  Per sweep
//   trace_q = trace1_q + sum_p T[q][p] (phi_in[p] - phi0[p])
//   upd_q   = gamma (g_q - trace_q);  phi_out[q] = phi_in[q] + upd_q
// T's columns are split three ways: [0, Creg) live in registers (K per
// thread, first row tile), [Creg, Creg + Cs) in shared memory, the rest is
// streamed from L2 (column segments of R rows are contiguous in the
// column-major layout).  The densities ping-pong between A and B: sweep idx
// reads A (idx odd) or B (idx even).  The sweep's max |update| goes to slot
// idx % 3 (block 0 clears slot (idx+1) % 3), one grid barrier, then every
// CTA reads the same max and takes the same decision.
struct OpSolveArgs {
  int n, first_idx, max_iter;
  double gamma, tol;
  RichState *st;
  double *history;
  unsigned long long *slots;      // [3]
  unsigned int *bar;              // grid barrier counter, zero at launch
  int rows;                       // R, rows per CTA
  int smem_cols;                  // Cs
};

// Grid barrier of the cooperative sweep kernels (all CTAs co-resident): a
// monotonically increasing arrival counter, release on arrival, acquire on
// the spin; thread 0 then reads the sweep's max |update| into *res.
// (~1.26 us per barrier on 148 CTAs against 1.67 us for cg::grid_group::sync,
// tools/mb/gsync.cu.)
KFBI_DEV void op_barrier(const OpSolveArgs &a, int sweep, double *res) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int target = (unsigned int)(sweep - a.first_idx + 1) * gridDim.x;
    unsigned int v;
    __threadfence();
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(a.bar) : "memory");
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    } while (v < target);
    *res = __longlong_as_double((long long)__ldcg(&a.slots[sweep % 3]));
  }
  __syncthreads();
}

constexpr int OP_THREADS = 512;
constexpr int OP_WARPS = OP_THREADS / 32;
template <typename T>
struct OpTune;                    // register cache K and streamed loads in flight U
#ifndef KFBI_OP_K_F64
#define KFBI_OP_K_F64 24
#endif
#ifndef KFBI_OP_K_HALF
#define KFBI_OP_K_HALF 12
#endif
template <> struct OpTune<double> { static constexpr int K = KFBI_OP_K_F64, U = 16; };
template <> struct OpTune<double2> { static constexpr int K = 12, U = 8; };

template <typename T>
inline size_t op_smem_fixed(int n) {
  return ((size_t)((n + 1) & ~1) + OP_WARPS * 32) * sizeof(T);
}

template <typename T, int K>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_solve_kernel(OpSolveArgs a, const T *__restrict__ Tcm, T *A, T *B,
                const T *__restrict__ phi0, const T *__restrict__ trace1,
                const T *__restrict__ g) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  T *d = reinterpret_cast<T *>(op_smem);                 // phi_in - phi0, [n]
  T *part = d + ((n + 1) & ~1);                          // [OP_WARPS][32]
  T *cache = part + OP_WARPS * 32;                       // [Cs][R], column-major
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const int creg = min(n, OP_WARPS * K);
  const int cs0 = creg, cg0 = min(n, creg + Cs);

  T treg[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int c = warp + OP_WARPS * k;
    treg[k] = (lane < nr && c < creg) ? Tcm[(size_t)c * n + r0 + lane] : S::zero();
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : S::zero();
  }
  if (a.st->done) return;                       // uniform: set before launch

  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const T *in = (idx & 1) ? A : B;
    T *out = (idx & 1) ? B : A;
    // d = phi_in - phi0: all of a thread's loads in flight at once (a
    // dependent loop of L2 round trips dominated the sweep before)
    for (int p0 = tid; p0 < n; p0 += OP_THREADS * 4) {
      T vi[4], v0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = p0 + u * OP_THREADS;
        vi[u] = p < n ? __ldcg(in + p) : S::zero();
        v0[u] = p < n ? __ldg(phi0 + p) : S::zero();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = p0 + u * OP_THREADS;
        if (p < n) d[p] = S::sub(vi[u], v0[u]);
      }
    }
    __syncthreads();
    double mag = 0.0;
    for (int rt = 0; rt < nr; rt += 32) {       // row tiles (one unless R > 32)
      const int row = rt + lane;
      const bool rok = row < nr;
      T acc = S::zero();
      if (rt == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int c = warp + OP_WARPS * k;
          if (c < creg) acc = S::add(acc, S::mul(treg[k], d[c]));
        }
      }
      if (rok)
        for (int c = cs0 + warp; c < cg0; c += OP_WARPS)
          acc = S::add(acc, S::mul(cache[(size_t)(c - cs0) * R + row], d[c]));
      constexpr int U = OpTune<T>::U;
      for (int c = cg0 + warp; c < n; c += OP_WARPS * U) {
        T v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int cc = c + OP_WARPS * u;
          v[u] = (rok && cc < n) ? __ldcg(Tcm + (size_t)cc * n + r0 + row) : S::zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int cc = c + OP_WARPS * u;
          if (cc < n) acc = S::add(acc, S::mul(v[u], d[cc]));
        }
      }
      part[warp * 32 + lane] = acc;
      __syncthreads();
      if (tid < 32 && rt + tid < nr) {
        const int q = r0 + rt + tid;
        T s = part[tid];
        for (int w = 1; w < OP_WARPS; ++w) s = S::add(s, part[w * 32 + tid]);
        const T trace = S::add(trace1[q], s);
        const T upd = S::rmul(S::sub(g[q], trace), a.gamma);
        out[q] = S::add(__ldcg(in + q), upd);
        mag = nanmax(mag, S::abs(upd));
      }
      __syncthreads();
    }
    if (warp == 0) {
      mag = warp_nanmax(mag);
      if (lane == 0) {
        atomic_max_nonneg(&a.slots[idx % 3], mag);
        if (blockIdx.x == 0) a.slots[(idx + 1) % 3] = 0ull;
      }
    }
    // one L2 read of the max per block (an atomic per thread would serialise)
    op_barrier(a, idx, &res_s);
    const double res = res_s;
    const bool conv = res <= a.tol;
    const bool last = conv || idx + 1 >= a.max_iter;
    if (blockIdx.x == 0 && tid == 0) {
      a.history[idx] = res;
      a.st->iters = idx + 1;
      a.st->last_res = res;
      if (conv) a.st->done = 1;
      else if (idx + 1 >= a.max_iter) a.st->done = 2;
    }
    if (last) break;
  }
}

// Small n_ctl (the latency path of small grids, C1: n = 88): every sweep
// inside ONE CTA, T transposed into shared memory (row-major: a warp reads
// one row's columns conflict free), the iterates ping-pong in shared memory,
// no grid barrier (1.3 us per sweep on the cooperative kernels, more than the
// sweep's work at this size).  Same sweep semantics and state protocol as
// op_solve_kernel: each sweep's iterate also goes to A / B by parity (the
// finaliser reads the last two), the history and RichState as there.
constexpr int OPC_THREADS = 1024;
template <typename T>
inline size_t op_cta_smem(int n) {
  return ((size_t)n * n + 6 * (size_t)n) * sizeof(T);
}

template <typename T>
__global__ void __launch_bounds__(OPC_THREADS, 1)
op_solve_cta_kernel(OpSolveArgs a, const T *__restrict__ Tcm, T *A, T *B,
                    const T *__restrict__ phi0, const T *__restrict__ trace1,
                    const T *__restrict__ g) {
  using S = Sc<T>;
  extern __shared__ __align__(16) unsigned char opc_smem[];
  __shared__ double wmax[OPC_THREADS / 32];
  const int n = a.n;
  T *Ts = reinterpret_cast<T *>(opc_smem);               // [n][n], Ts[q n + c] = T(q, c)
  T *ph = Ts + (size_t)n * n;                            // [2][n] iterates
  T *d = ph + 2 * n, *p0 = d + n, *t1 = p0 + n, *gs = t1 + n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.st->done) return;                       // uniform: set before launch
  for (int i = tid; i < n * n; i += OPC_THREADS) {   // Ts[q n + c] = Tcm[c n + q]
    const int q = i / n, c = i - q * n;
    Ts[i] = __ldg(&Tcm[(size_t)c * n + q]);
  }
  for (int i = tid; i < n; i += OPC_THREADS) {
    p0[i] = phi0[i];
    t1[i] = trace1[i];
    gs[i] = g[i];
    ph[((a.first_idx & 1) ^ 1) * n + i] = (a.first_idx & 1) ? A[i] : B[i];   // the first input
  }
  __syncthreads();
  // 8 lanes per row (four rows per warp at once), shuffle sums within the
  // group; the sweep max by one warp
  constexpr int GL = 8;
  const int sub = lane & (GL - 1), grp = tid / GL;
  constexpr int NG = OPC_THREADS / GL;
  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const T *in = ph + ((idx & 1) ^ 1) * n;     // A-side iterate for odd idx (as op_solve_kernel)
    T *outs = ph + (idx & 1) * n;
    T *outg = (idx & 1) ? B : A;
    for (int i = tid; i < n; i += OPC_THREADS) d[i] = S::sub(in[i], p0[i]);
    __syncthreads();
    double mag = 0.0;
    for (int q0 = 0; q0 < n; q0 += NG) {
      const int q = q0 + grp;
      T acc = S::zero();
      if (q < n) {
        const T *row = Ts + (size_t)q * n;
        for (int c = sub; c < n; c += GL) acc = S::add(acc, S::mul(row[c], d[c]));
      }
#pragma unroll
      for (int off = GL / 2; off >= 1; off >>= 1) {
        if constexpr (std::is_same<T, double>::value) acc += __shfl_down_sync(0xffffffffu, acc, off, GL);
        else {
          acc.x += __shfl_down_sync(0xffffffffu, acc.x, off, GL);
          acc.y += __shfl_down_sync(0xffffffffu, acc.y, off, GL);
        }
      }
      if (sub == 0 && q < n) {
        const T trace = S::add(t1[q], acc);
        const T upd = S::rmul(S::sub(gs[q], trace), a.gamma);
        const T o = S::add(in[q], upd);
        outs[q] = o;
        outg[q] = o;
        mag = nanmax(mag, S::abs(upd));
      }
    }
    mag = warp_nanmax(mag);
    if (lane == 0) wmax[warp] = mag;
    __syncthreads();
    if (warp == 0) {
      double v = warp_nanmax(wmax[lane]);
      if (lane == 0) wmax[0] = v;
    }
    __syncthreads();
    const double res = wmax[0];
    const bool conv = res <= a.tol;
    const bool last = conv || idx + 1 >= a.max_iter;
    if (tid == 0) {
      a.history[idx] = res;
      a.st->iters = idx + 1;
      a.st->last_res = res;
      if (conv) a.st->done = 1;
      else if (idx + 1 >= a.max_iter) a.st->done = 2;
    }
    __syncthreads();                            // wmax / d reused by the next sweep
    if (last) break;
  }
}

// f64 operator sweeps with two rows per lane: half-warp h of warp w works on
// columns 2w + h + 32 s, lane l of the half on rows (2l, 2l+1) of the CTA's
// block, so every shared-memory and global load of T is a 16-byte pair and
// each instruction covers two columns (half the instructions of the one-row
// kernel above, which remains the complex / odd-n path).  Same sweep
// semantics, same convergence protocol.  Requires n and R even.
template <int K2, int G>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_solve_pair_kernel(OpSolveArgs a, const double *__restrict__ Tcm, double *A, double *B,
                     const double *__restrict__ phi0, const double *__restrict__ trace1,
                     const double *__restrict__ g) {
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  double *d = reinterpret_cast<double *>(op_smem);       // phi_in - phi0, [n]
  double *part = d + ((n + 1) & ~1);                     // [OP_WARPS][32]
  double *cache = part + OP_WARPS * 32;                  // [Cs][R], column-major
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // G column groups per warp, RPL = 32 / G row pairs per group: lane l is
  // row pair hl of group hf (G = 2: half-warps; G = 3: 10 pairs, lanes 30-31 idle)
  constexpr int RPL = 32 / G;
  const int hf = lane / RPL, hl = lane - hf * RPL;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const bool rok = hf < G && 2 * hl < nr;
  const int creg = min(n, G * OP_WARPS * K2);
  const int cs0 = creg, cg0 = min(n, creg + Cs);
  const int c_off = G * warp + hf;                       // first column of this lane group
  constexpr int PD = 8;                                  // d entries per thread and round
  double p0r[PD];                                        // phi0 of the first round, kept
#pragma unroll
  for (int u = 0; u < PD; ++u) {
    const int p = tid + u * OP_THREADS;
    p0r[u] = p < n ? phi0[p] : 0.0;
  }

  double2 treg[K2];
#pragma unroll
  for (int k = 0; k < K2; ++k) {
    const int c = c_off + G * OP_WARPS * k;
    treg[k] = (rok && c < creg) ? *reinterpret_cast<const double2 *>(Tcm + (size_t)c * n + r0 + 2 * hl)
                                : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : 0.0;
  }
  if (a.st->done) return;                       // uniform: set before launch

  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const double *in = (idx & 1) ? A : B;
    double *out = (idx & 1) ? B : A;
    // all of a thread's d loads in one round (n <= 4096: one L2 round trip)
    for (int q0 = 0; q0 < n; q0 += OP_THREADS * PD) {
      double vi[PD];
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        vi[u] = p < n ? __ldcg(in + p) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < PD; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        if (p < n) d[p] = vi[u] - (q0 == 0 ? p0r[u] : __ldg(phi0 + p));
      }
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const int c = c_off + G * OP_WARPS * k;
      if (rok && c < creg) {
        const double dc = d[c];
        acc.x = fma(treg[k].x, dc, acc.x);
        acc.y = fma(treg[k].y, dc, acc.y);
      }
    }
    if (rok)
      for (int c = cs0 + c_off; c < cg0; c += G * OP_WARPS) {
        const double2 t2 = *reinterpret_cast<const double2 *>(cache + (size_t)(c - cs0) * R + 2 * hl);
        const double dc = d[c];
        acc.x = fma(t2.x, dc, acc.x);
        acc.y = fma(t2.y, dc, acc.y);
      }
    constexpr int U = 8;
    for (int c = cg0 + c_off; c < n; c += G * OP_WARPS * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + G * OP_WARPS * u;
        v[u] = (rok && cc < n)
                   ? __ldcg(reinterpret_cast<const double2 *>(Tcm + (size_t)cc * n + r0 + 2 * hl))
                   : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + G * OP_WARPS * u;
        if (cc < n) {
          const double dc = d[cc];
          acc.x = fma(v[u].x, dc, acc.x);
          acc.y = fma(v[u].y, dc, acc.y);
        }
      }
    }
    // the G column groups of the warp hold partial sums of the same rows
    if constexpr (G == 2) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
    } else {
      double2 tot = acc;
#pragma unroll
      for (int gg = 1; gg < G; ++gg) {
        const int src = min(lane + gg * RPL, 31);
        tot.x += __shfl_sync(0xffffffffu, acc.x, src);
        tot.y += __shfl_sync(0xffffffffu, acc.y, src);
      }
      acc = tot;
    }
    if (hf == 0) {
      part[warp * 32 + 2 * hl] = acc.x;
      part[warp * 32 + 2 * hl + 1] = acc.y;
    }
    __syncthreads();
    double mag = 0.0;
    if (tid < 32 && tid < nr) {
      const int q = r0 + tid;
      double s2 = part[tid];
      for (int w = 1; w < OP_WARPS; ++w) s2 += part[w * 32 + tid];
      const double trace = trace1[q] + s2;
      const double upd = (g[q] - trace) * a.gamma;
      out[q] = __ldcg(in + q) + upd;
      mag = fabs(upd);
    }
    if (warp == 0) {
      mag = warp_nanmax(mag);
      if (lane == 0) {
        atomic_max_nonneg(&a.slots[idx % 3], mag);
        if (blockIdx.x == 0) a.slots[(idx + 1) % 3] = 0ull;
      }
    }
    op_barrier(a, idx, &res_s);
    const double res = res_s;
    const bool conv = res <= a.tol;
    const bool last = conv || idx + 1 >= a.max_iter;
    if (blockIdx.x == 0 && tid == 0) {
      a.history[idx] = res;
      a.st->iters = idx + 1;
      a.st->last_res = res;
      if (conv) a.st->done = 1;
      else if (idx + 1 >= a.max_iter) a.st->done = 2;
    }
    if (last) break;
  }
}

// c128 operator sweeps for R <= 16 rows per CTA: half-warp h of warp w works
// on columns 2w + h + 32 s, lane l of the half on row l (one 16-byte complex),
// so 16 lanes stay busy where the one-row-per-lane kernel above keeps R of 32.
// Same accumulation order per row as op_solve_kernel<double2> (register,
// shared, streamed columns in increasing order within a lane's column set);
// same sweep semantics and convergence protocol.
template <int K>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_solve_half_kernel(OpSolveArgs a, const double2 *__restrict__ Tcm, double2 *A, double2 *B,
                     const double2 *__restrict__ phi0, const double2 *__restrict__ trace1,
                     const double2 *__restrict__ g) {
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  double2 *d = reinterpret_cast<double2 *>(op_smem);     // phi_in - phi0, [n]
  double2 *part = d + ((n + 1) & ~1);                    // [OP_WARPS][32]
  double2 *cache = part + OP_WARPS * 32;                 // [Cs][R], column-major
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hl = lane & 15, hf = lane >> 4;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const bool rok = hl < nr;
  const int creg = min(n, 2 * OP_WARPS * K);
  const int cs0 = creg, cg0 = min(n, creg + Cs);
  const int c_off = 2 * warp + hf;
  double2 treg[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int c = c_off + 2 * OP_WARPS * k;
    treg[k] = (rok && c < creg) ? Tcm[(size_t)c * n + r0 + hl] : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : make_double2(0.0, 0.0);
  }
  if (a.st->done) return;
  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const double2 *in = (idx & 1) ? A : B;
    double2 *out = (idx & 1) ? B : A;
    for (int q0 = 0; q0 < n; q0 += OP_THREADS * 4) {
      double2 vi[4], v0[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        vi[u] = p < n ? __ldcg(in + p) : make_double2(0.0, 0.0);
        v0[u] = p < n ? __ldg(phi0 + p) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        if (p < n) d[p] = csub(vi[u], v0[u]);
      }
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = c_off + 2 * OP_WARPS * k;
      if (c < creg) acc = cadd(acc, cmul(treg[k], d[c]));
    }
    if (rok)
      for (int c = cs0 + c_off; c < cg0; c += 2 * OP_WARPS)
        acc = cadd(acc, cmul(cache[(size_t)(c - cs0) * R + hl], d[c]));
    constexpr int U = 8;
    for (int c = cg0 + c_off; c < n; c += 2 * OP_WARPS * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + 2 * OP_WARPS * u;
        v[u] = (rok && cc < n) ? __ldcg(Tcm + (size_t)cc * n + r0 + hl) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + 2 * OP_WARPS * u;
        if (cc < n) acc = cadd(acc, cmul(v[u], d[cc]));
      }
    }
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
    if (hf == 0) part[warp * 32 + hl] = acc;
    __syncthreads();
    double mag = 0.0;
    if (tid < 32 && tid < nr) {
      const int q = r0 + tid;
      double2 s2 = part[tid];
      for (int w = 1; w < OP_WARPS; ++w) s2 = cadd(s2, part[w * 32 + tid]);
      const double2 trace = cadd(trace1[q], s2);
      const double2 upd = cscale(csub(g[q], trace), a.gamma);
      out[q] = cadd(__ldcg(in + q), upd);
      mag = hypot(upd.x, upd.y);
    }
    if (warp == 0) {
      mag = warp_nanmax(mag);
      if (lane == 0) {
        atomic_max_nonneg(&a.slots[idx % 3], mag);
        if (blockIdx.x == 0) a.slots[(idx + 1) % 3] = 0ull;
      }
    }
    op_barrier(a, idx, &res_s);
    const double res = res_s;
    const bool conv = res <= a.tol;
    const bool last = conv || idx + 1 >= a.max_iter;
    if (blockIdx.x == 0 && tid == 0) {
      a.history[idx] = res;
      a.st->iters = idx + 1;
      a.st->last_res = res;
      if (conv) a.st->done = 1;
      else if (idx + 1 >= a.max_iter) a.st->done = 2;
    }
    if (last) break;
  }
}

// Extraction writing the BvpSolution traces (u+, d_n u+) of a final field.
template <typename T>
__global__ void __launch_bounds__(256)
extract_traces_kernel(ExtractArgs x, const T *__restrict__ u, const T *__restrict__ jm,
                      T *trace_u, T *trace_un, const int *skip) {
  using S = Sc<T>;
  if (skip && *skip) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= x.n) return;
  T tu, tx, ty;
  extract_any<T>(x, u, jm, p, tu, tx, ty);
  trace_u[p] = tu;
  trace_un[p] = S::add(S::rmul(tx, x.normal[2 * p]), S::rmul(ty, x.normal[2 * p + 1]));
}

// Per-step record of an asynchronous solve (read back in batches by the host).
struct StepLog {
  int iterations;
  int status;                     // 1 converged, 2 max_iter reached
  double residual;
  double norm;                    // blow-up norm of the step, when logged
  double newton;                  // worst pointwise Newton residual (Schrodinger)
};

// Closes an operator-form solve on the device, without the host:
//   K = sweeps done; skip[0] = 0 only if the converging sweep was an
//   operator sweep (then the full pipeline must recompute the field from
//   phi_(K-1)); phi_(K-1) -> phik1, phi_K -> A (ping-pong parity of
//   op_solve_kernel); the step log entry.
template <typename T>
__global__ void op_finalize_kernel(const RichState *st, int n, T *A, const T *B, T *phik1,
                                   int *skip, StepLog *log, const T *phi0 = nullptr) {
  // phi0 != null: sweep 1 formed only its trace, so a solve converging at
  // sweep 1 also needs the field, from phi_0
  const int K = st->iters, done = st->done;
  const bool odd = (K & 1) != 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    if (K >= 2) {
      const T a = A[p], b = B[p];
      phik1[p] = odd ? b : a;       // phi_(K-1)
      if (!odd) A[p] = b;           // phi_K into the density buffer
    } else if (phi0) {
      phik1[p] = phi0[p];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    skip[0] = ((K >= 2 || phi0) && done == 1) ? 0 : 1;
    if (log) {
      log->iterations = K;
      log->status = done;
      log->residual = st->last_res;
    }
  }
}

// dst = src while the Richardson solve runs: keeps phi_(K-1), the density the
// converging sweep started from (the pipeline form with trace-only sweeps)
template <typename T>
__global__ void copy_running_kernel(const RichState *st, int n, const T *src, T *dst) {
  if (st->done) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) dst[p] = src[p];
}

__global__ void log_norm_kernel(const unsigned long long *norm_bits, StepLog *log, int which) {
  const double v = __longlong_as_double((long long)*norm_bits);
  if (which == 0) log->norm = v;
  else log->newton = nanmax(log->newton, v);
}

__global__ void rich_init_kernel(RichState *st, int max_iter, double tol) {
  st->done = 0;
  st->iters = 0;
  st->max_iter = max_iter;
  st->tol = tol;
  st->last_res = 0.0;
  st->res_bits = 0ull;
  st->arrive = 0u;
}

}  // namespace kfbi
