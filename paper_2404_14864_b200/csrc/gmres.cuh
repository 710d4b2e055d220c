// Restarted GMRES on the boundary integral equation (opt-in alternative to
// the damped Richardson iteration of bvp.py:276-351; PAPER.md:768 and
// SPEC.md:349 name Krylov solvers as the follow-up).
//
// The sweep map phi -> trace(phi) is affine (bvp.py:312-323): trace(phi) =
// t_F + T phi with T the trace operator of the geometry and kappa.  Richardson
// iterates phi <- phi + gamma (g - trace(phi)); GMRES solves T phi = g - t_F
// directly: r0 = g - trace(phi0) from one full sweep, Krylov vectors from
// matvecs T v (the pipeline with F = 0, f_gamma = 0, or the plan's explicit
// trace operator), classical Gram-Schmidt applied twice, Givens rotations.
// Everything stays on the device: the kernels below are guarded by the state's
// `done` flag, so a whole restart cycle is enqueued without host round trips.
// Stopping rule: gamma * ||g - trace(phi)||_2 <= tol, which implies the
// reference's max-norm criterion on the update gamma (g - trace).
#pragma once

#include "common.cuh"

namespace kfbi {

struct GmresState {
  int done;                 // 0 running, 1 converged, 2 max_iter (guarded kernels skip)
  int iters;                // matvecs so far (all cycles)
  int k;                    // Arnoldi steps completed in the current cycle
  int max_iter;
  double tol, gamma;
  double resid;             // ||g - trace||_2 estimate (Givens)
  double inv;               // 1 / H[j+1, j] of the last step
  int full;                 // the cycle used all its steps
  int pad;
};

constexpr int GM_NB = 64;             // blocks of the reduction kernels
constexpr int GM_T = 256;

template <typename T> KFBI_DEV T gm_conj(T v);
template <> KFBI_DEV double gm_conj<double>(double v) { return v; }
template <> KFBI_DEV double2 gm_conj<double2>(double2 v) { return cconj(v); }
KFBI_DEV double gm_abs2(double v) { return v * v; }
KFBI_DEV double gm_abs2(double2 v) { return v.x * v.x + v.y * v.y; }

// block-wide sum of a T (fixed order: deterministic)
template <typename T>
KFBI_DEV T gm_block_sum(T v, T *scr) {
  using S = Sc<T>;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if constexpr (std::is_same<T, double>::value) v = warp_sum(v);
  else {
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
  }
  if (lane == 0) scr[w] = v;
  __syncthreads();
  T acc = S::zero();
  if (threadIdx.x == 0)
    for (int i = 0; i < GM_T / 32; ++i) acc = S::add(acc, scr[i]);
  __syncthreads();
  return acc;                         // valid in thread 0
}

// r = g - trace (cycle start), norm partials
template <typename T>
__global__ void __launch_bounds__(GM_T) gm_start_kernel(int n, const T *g, const T *trace, T *r,
                                                        double *npart, const GmresState *st) {
  __shared__ double scr[GM_T / 32];
  if (st->done) return;
  double acc = 0.0;
  for (int i = blockIdx.x * GM_T + threadIdx.x; i < n; i += GM_NB * GM_T) {
    const T v = Sc<T>::sub(g[i], trace[i]);
    r[i] = v;
    acc += gm_abs2(v);
  }
  const double s = gm_block_sum<double>(acc, scr);
  if (threadIdx.x == 0) npart[blockIdx.x] = s;
}

// beta = ||r||, gvec = (beta, 0, ...), cycle reset; converged already -> done
template <typename T>
__global__ void gm_begin_kernel(const double *npart, T *gvec, GmresState *st, double *history) {
  if (threadIdx.x != 0 || st->done) return;
  double s = 0.0;
  for (int b = 0; b < GM_NB; ++b) s += npart[b];
  const double beta = sqrt(s);
  gvec[0] = Sc<T>::rmul(Sc<T>::one(), beta);
  st->k = 0;
  st->full = 0;
  st->resid = beta;
  st->inv = beta > 0.0 ? 1.0 / beta : 0.0;
  if (st->gamma * beta <= st->tol) st->done = 1;
  (void)history;
}

// dst = src * st->inv
template <typename T>
__global__ void __launch_bounds__(GM_T) gm_scale_kernel(int n, const T *src, T *dst, const GmresState *st) {
  if (st->done) return;
  const double inv = st->inv;
  for (int i = blockIdx.x * GM_T + threadIdx.x; i < n; i += GM_NB * GM_T) dst[i] = Sc<T>::rmul(src[i], inv);
}

// partial dots <V_i, w> (conj(V_i) . w), i <= j
template <typename T>
__global__ void __launch_bounds__(GM_T) gm_dots_kernel(int n, int j, const T *V, const T *w, T *part,
                                                       const GmresState *st) {
  __shared__ T scr[GM_T / 32];
  if (st->done) return;
  for (int i = 0; i <= j; ++i) {
    const T *vi = V + (size_t)i * n;
    T acc = Sc<T>::zero();
    for (int q = blockIdx.x * GM_T + threadIdx.x; q < n; q += GM_NB * GM_T)
      acc = Sc<T>::add(acc, Sc<T>::mul(gm_conj<T>(vi[q]), w[q]));
    const T s = gm_block_sum<T>(acc, scr);
    if (threadIdx.x == 0) part[(size_t)i * GM_NB + blockIdx.x] = s;
  }
}

// h_i = sum of the partials (every block, fixed order); H[:, j] (+)= h;
// w -= sum_i h_i V_i; norm partials of the new w
template <typename T>
__global__ void __launch_bounds__(GM_T) gm_orth_kernel(int n, int j, int m, const T *V, T *w,
                                                       const T *part, T *H, int accumulate,
                                                       double *npart, const GmresState *st) {
  __shared__ T h[65];
  __shared__ double scr[GM_T / 32];
  if (st->done) return;
  for (int i = threadIdx.x; i <= j; i += GM_T) {
    T s = Sc<T>::zero();
    for (int b = 0; b < GM_NB; ++b) s = Sc<T>::add(s, part[(size_t)i * GM_NB + b]);
    h[i] = s;
    if (blockIdx.x == 0) H[(size_t)i * m + j] = accumulate ? Sc<T>::add(H[(size_t)i * m + j], s) : s;
  }
  __syncthreads();
  double acc = 0.0;
  for (int q = blockIdx.x * GM_T + threadIdx.x; q < n; q += GM_NB * GM_T) {
    T v = w[q];
    for (int i = 0; i <= j; ++i) v = Sc<T>::sub(v, Sc<T>::mul(h[i], V[(size_t)i * n + q]));
    w[q] = v;
    acc += gm_abs2(v);
  }
  const double s = gm_block_sum<double>(acc, scr);
  if (threadIdx.x == 0) npart[blockIdx.x] = s;
}

// H[j+1, j] = ||w||; earlier rotations on column j; a new rotation zeroes
// H[j+1, j]; residual |gvec[j+1]|; convergence.
template <typename T>
__global__ void gm_givens_kernel(int j, int m, const double *npart, T *H, double *cs, T *sn, T *gvec,
                                 GmresState *st, double *history) {
  using S = Sc<T>;
  if (threadIdx.x != 0 || st->done) return;
  double s2 = 0.0;
  for (int b = 0; b < GM_NB; ++b) s2 += npart[b];
  const double hn = sqrt(s2);
  for (int i = 0; i < j; ++i) {                  // apply G_i to rows i, i+1 of column j
    const T a = H[(size_t)i * m + j], b = H[(size_t)(i + 1) * m + j];
    H[(size_t)i * m + j] = S::add(S::rmul(a, cs[i]), S::mul(sn[i], b));
    H[(size_t)(i + 1) * m + j] = S::sub(S::rmul(b, cs[i]), S::mul(gm_conj<T>(sn[i]), a));
  }
  const T a = H[(size_t)j * m + j];
  const double aa = sqrt(gm_abs2(a));
  const double rr = sqrt(aa * aa + hn * hn);
  double c;
  T s;
  if (aa == 0.0) {
    c = 0.0;
    s = S::one();
  } else {
    c = aa / rr;
    s = S::rmul(a, hn / (aa * rr));              // (a / |a|) conj(b) / r, b = hn real
  }
  cs[j] = c;
  sn[j] = s;
  H[(size_t)j * m + j] = aa == 0.0 ? S::rmul(S::one(), hn) : S::rmul(a, rr / aa);
  const T gj = gvec[j];
  gvec[j] = S::rmul(gj, c);
  const T gn = S::sub(S::zero(), S::mul(gm_conj<T>(s), gj));
  gvec[j + 1] = gn;
  const double res = sqrt(gm_abs2(gn));
  const int it = st->iters + 1;
  if (it - 1 < st->max_iter) history[it - 1] = st->gamma * res;
  st->iters = it;
  st->k = j + 1;
  st->resid = res;
  st->inv = hn > 0.0 ? 1.0 / hn : 0.0;
  if (st->gamma * res <= st->tol || hn == 0.0) st->done = 1;
  else if (it >= st->max_iter) st->done = 2;
  else if (j + 1 == m) st->full = 1;
}

// y = R^{-1} gvec[0:k] (upper triangular H), x += V y   (one block, then all)
template <typename T>
__global__ void gm_backsolve_kernel(int m, const T *H, const T *gvec, T *y, const GmresState *st) {
  using S = Sc<T>;
  if (threadIdx.x != 0) return;
  const int k = st->k;
  for (int i = k - 1; i >= 0; --i) {
    T v = gvec[i];
    for (int q = i + 1; q < k; ++q) v = S::sub(v, S::mul(H[(size_t)i * m + q], y[q]));
    const T d = H[(size_t)i * m + i];
    if constexpr (std::is_same<T, double>::value) y[i] = v / d;
    else y[i] = cdiv(v, d);
  }
}

template <typename T>
__global__ void __launch_bounds__(GM_T) gm_update_kernel(int n, const T *V, const T *y, T *x,
                                                         const GmresState *st) {
  const int k = st->k;
  for (int q = blockIdx.x * GM_T + threadIdx.x; q < n; q += GM_NB * GM_T) {
    T v = x[q];
    for (int i = 0; i < k; ++i) v = Sc<T>::add(v, Sc<T>::mul(y[i], V[(size_t)i * n + q]));
    x[q] = v;
  }
}

// y = Top v (column-major n x n trace operator), partial over column slices
constexpr int GM_JS = 16;
template <typename T>
__global__ void __launch_bounds__(GM_T) gm_gemv_kernel(int n, const T *Top, const T *v, T *part,
                                                       const GmresState *st) {
  if (st->done) return;
  const int i = blockIdx.x * GM_T + threadIdx.x;
  if (i >= n) return;
  const int c0 = (int)((long)n * blockIdx.y / GM_JS), c1 = (int)((long)n * (blockIdx.y + 1) / GM_JS);
  T acc = Sc<T>::zero();
  for (int c = c0; c < c1; ++c) acc = Sc<T>::add(acc, Sc<T>::mul(Top[(size_t)c * n + i], v[c]));
  part[(size_t)blockIdx.y * n + i] = acc;
}

template <typename T>
__global__ void __launch_bounds__(GM_T) gm_gemv_sum_kernel(int n, const T *part, T *w, const GmresState *st) {
  if (st->done) return;
  const int i = blockIdx.x * GM_T + threadIdx.x;
  if (i >= n) return;
  T acc = Sc<T>::zero();
  for (int s = 0; s < GM_JS; ++s) acc = Sc<T>::add(acc, part[(size_t)s * n + i]);
  w[i] = acc;
}

__global__ void gm_init_kernel(GmresState *st, int max_iter, double tol, double gamma) {
  st->done = 0;
  st->iters = 0;
  st->k = 0;
  st->max_iter = max_iter;
  st->tol = tol;
  st->gamma = gamma;
  st->resid = 0.0;
  st->inv = 0.0;
  st->full = 0;
}

}  // namespace kfbi
