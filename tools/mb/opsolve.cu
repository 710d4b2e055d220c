// Microbenchmark of the operator-form sweep kernel (op_solve_pair_kernel):
// random T (n x n, column-major), tol = 0 so every launch runs max_iter
// sweeps; prints us per sweep and a checksum of the final density.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2404_14864_b200/csrc \
//        -o tools/mb/opsolve tools/mb/opsolve.cu && tools/mb/opsolve 2850 3800
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "interface_kernels.cuh"

using namespace kfbi;

// ---- variant: phi0 in registers, one-round d load, streamed batch
// prefetched across the barrier (PREF), hand-rolled barrier (BAR) ----
template <int K2, int U, bool PREF, bool BAR>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_pair_v(OpSolveArgs a, const double *__restrict__ Tcm, double *A, double *B,
          const double *__restrict__ phi0, const double *__restrict__ trace1,
          const double *__restrict__ g, unsigned int *ctr) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  double *d = reinterpret_cast<double *>(op_smem);
  double *part = d + ((n + 1) & ~1);
  double *cache = part + OP_WARPS * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hl = lane & 15, hf = lane >> 4;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const bool rok = 2 * hl < nr;
  const int creg = min(n, 2 * OP_WARPS * K2);
  const int cs0 = creg, cg0 = min(n, creg + Cs);
  const int c_off = 2 * warp + hf;
  constexpr int PD = 8;                     // d entries per thread (n <= 4096 in one round)
  double p0r[PD];
#pragma unroll
  for (int u = 0; u < PD; ++u) {
    const int p = tid + u * OP_THREADS;
    p0r[u] = p < n ? phi0[p] : 0.0;
  }
  double2 treg[K2];
#pragma unroll
  for (int k = 0; k < K2; ++k) {
    const int c = c_off + 2 * OP_WARPS * k;
    treg[k] = (rok && c < creg) ? *reinterpret_cast<const double2 *>(Tcm + (size_t)c * n + r0 + 2 * hl)
                                : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : 0.0;
  }
  if (a.st->done) return;
  double2 pre[U];
  auto load_batch = [&](int c, double2 (&v)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int cc = c + 2 * OP_WARPS * u;
      v[u] = (rok && cc < n) ? __ldcg(reinterpret_cast<const double2 *>(Tcm + (size_t)cc * n + r0 + 2 * hl))
                             : make_double2(0.0, 0.0);
    }
  };
  if (PREF) load_batch(cg0 + c_off, pre);
  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const double *in = (idx & 1) ? A : B;
    double *out = (idx & 1) ? B : A;
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
        if (p < n) d[p] = vi[u] - (q0 == 0 ? p0r[u] : phi0[p]);
      }
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const int c = c_off + 2 * OP_WARPS * k;
      if (c < creg) {
        const double dc = d[c];
        acc.x = fma(treg[k].x, dc, acc.x);
        acc.y = fma(treg[k].y, dc, acc.y);
      }
    }
    if (rok)
      for (int c = cs0 + c_off; c < cg0; c += 2 * OP_WARPS) {
        const double2 t2 = *reinterpret_cast<const double2 *>(cache + (size_t)(c - cs0) * R + 2 * hl);
        const double dc = d[c];
        acc.x = fma(t2.x, dc, acc.x);
        acc.y = fma(t2.y, dc, acc.y);
      }
    for (int c = cg0 + c_off; c < n; c += 2 * OP_WARPS * U) {
      double2 v[U];
      if (PREF && c == cg0 + c_off) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = pre[u];
      } else {
        load_batch(c, v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + 2 * OP_WARPS * u;
        if (cc < n) {
          const double dc = d[cc];
          acc.x = fma(v[u].x, dc, acc.x);
          acc.y = fma(v[u].y, dc, acc.y);
        }
      }
    }
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
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
    if (PREF) load_batch(cg0 + c_off, pre);
    if (BAR) {
      __syncthreads();
      if (tid == 0) {
        const unsigned int target = (unsigned int)(idx - a.first_idx + 1) * gridDim.x;
        unsigned int v;
        __threadfence();
        asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
        do {
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
        res_s = __longlong_as_double((long long)__ldcg(&a.slots[idx % 3]));
      }
      __syncthreads();
    } else {
      grid.sync();
      if (tid == 0) res_s = __longlong_as_double((long long)__ldcg(&a.slots[idx % 3]));
      __syncthreads();
    }
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


// ---- variant: streamed part through a cp.async ring in shared memory
// (thread-private slots, no registers held by loads in flight); the first
// NS-1 stages of the next sweep are issued before the barrier ----
KFBI_DEV void cp16(void *smem_dst, const void *gsrc, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gsrc), "r"(sz) : "memory");
}
KFBI_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
KFBI_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int K2, int UB, int NS, bool PREF>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_pair_ca(OpSolveArgs a, const double *__restrict__ Tcm, double *A, double *B,
           const double *__restrict__ phi0, const double *__restrict__ trace1,
           const double *__restrict__ g, unsigned int *ctr) {
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  double2 *ring = reinterpret_cast<double2 *>(op_smem);                 // [NS][UB][OP_THREADS]
  double *d = reinterpret_cast<double *>(ring + NS * UB * OP_THREADS);
  double *part = d + ((n + 1) & ~1);
  double *cache = part + OP_WARPS * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hl = lane & 15, hf = lane >> 4;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const bool rok = 2 * hl < nr;
  const int creg = min(n, 2 * OP_WARPS * K2);
  const int cs0 = creg, cg0 = min(n, creg + Cs);
  const int c_off = 2 * warp + hf;
  constexpr int CST = 2 * OP_WARPS;                     // column step of one load
  const int nst = (n - cg0 + CST * UB - 1) / (CST * UB); // stages per sweep (uniform)
  double2 treg[K2];
#pragma unroll
  for (int k = 0; k < K2; ++k) {
    const int c = c_off + 2 * OP_WARPS * k;
    treg[k] = (rok && c < creg) ? *reinterpret_cast<const double2 *>(Tcm + (size_t)c * n + r0 + 2 * hl)
                                : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : 0.0;
  }
  if (a.st->done) return;
  auto issue = [&](int stg) {                            // stage stg of the sweep
    if (stg < nst) {
      double2 *slot = ring + (stg % NS) * UB * OP_THREADS + tid;
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int cc = cg0 + c_off + CST * (stg * UB + u);
        const bool ok = rok && cc < n;
        cp16(slot + u * OP_THREADS, ok ? (const void *)(Tcm + (size_t)cc * n + r0 + 2 * hl) : (const void *)Tcm, ok);
      }
    }
    cp_commit();
  };
  if (PREF)
    for (int st = 0; st < NS - 1; ++st) issue(st);
  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const double *in = (idx & 1) ? A : B;
    double *out = (idx & 1) ? B : A;
    if (!PREF)
      for (int st = 0; st < NS - 1; ++st) issue(st);
    for (int q0 = 0; q0 < n; q0 += OP_THREADS * 8) {
      double vi[8], v0[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        vi[u] = p < n ? __ldcg(in + p) : 0.0;
        v0[u] = p < n ? __ldg(phi0 + p) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        if (p < n) d[p] = vi[u] - v0[u];
      }
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const int c = c_off + 2 * OP_WARPS * k;
      if (c < creg) {
        const double dc = d[c];
        acc.x = fma(treg[k].x, dc, acc.x);
        acc.y = fma(treg[k].y, dc, acc.y);
      }
    }
    if (rok)
      for (int c = cs0 + c_off; c < cg0; c += 2 * OP_WARPS) {
        const double2 t2 = *reinterpret_cast<const double2 *>(cache + (size_t)(c - cs0) * R + 2 * hl);
        const double dc = d[c];
        acc.x = fma(t2.x, dc, acc.x);
        acc.y = fma(t2.y, dc, acc.y);
      }
    for (int stg = 0; stg < nst; ++stg) {
      issue(stg + NS - 1);
      cp_wait<NS - 1>();
      const double2 *slot = ring + (stg % NS) * UB * OP_THREADS + tid;
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int cc = cg0 + c_off + CST * (stg * UB + u);
        if (cc < n) {
          const double2 v = slot[u * OP_THREADS];
          const double dc = d[cc];
          acc.x = fma(v.x, dc, acc.x);
          acc.y = fma(v.y, dc, acc.y);
        }
      }
    }
    cp_wait<0>();
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
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
    if (PREF)
      for (int st = 0; st < NS - 1; ++st) issue(st);
    __syncthreads();
    if (tid == 0) {
      const unsigned int target = (unsigned int)(idx - a.first_idx + 1) * gridDim.x;
      unsigned int v;
      __threadfence();
      asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(ctr) : "memory");
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
      res_s = __longlong_as_double((long long)__ldcg(&a.slots[idx % 3]));
    }
    __syncthreads();
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
  cp_wait<0>();
}


// ---- variant: barrier-free sweeps.  Each CTA publishes its new densities
// and its local max |update| as LL words (32-bit epoch + 32-bit half of the
// value, one 64-bit store each, so every word is single-copy atomic); the
// next sweep's readers poll the words until the epoch matches.  Two buffers
// by sweep parity (a CTA can be at most one sweep ahead of any other). ----
KFBI_DEV unsigned long long ll_word(unsigned int half, unsigned int epoch) {
  return ((unsigned long long)half << 32) | epoch;
}
KFBI_DEV void ll_put(unsigned long long *w, double v, unsigned int epoch) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ll_word((unsigned int)(b >> 32), epoch), w1 = ll_word((unsigned int)b, epoch);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(w), "l"(w0), "l"(w1) : "memory");
}
// poll until both words carry `epoch` (bounded; returns false on timeout)
KFBI_DEV bool ll_get(const unsigned long long *w, unsigned int epoch, double &v) {
  for (int it = 0; it < (1 << 22); ++it) {
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(w) : "memory");
    if ((unsigned int)w0 == epoch && (unsigned int)w1 == epoch) {
      v = __longlong_as_double((long long)((w0 & 0xffffffff00000000ull) | (w1 >> 32)));
      return true;
    }
  }
  return false;
}

template <int K2, int U>
__global__ void __launch_bounds__(OP_THREADS, 1)
op_pair_ll(OpSolveArgs a, const double *__restrict__ Tcm, double *A, double *B,
           const double *__restrict__ phi0, const double *__restrict__ trace1,
           const double *__restrict__ g, unsigned long long *ll, unsigned int ebase) {
  extern __shared__ __align__(16) unsigned char op_smem[];
  __shared__ double res_w[OP_WARPS];
  __shared__ int bad_s;
  const int n = a.n, R = a.rows, Cs = a.smem_cols;
  double *d = reinterpret_cast<double *>(op_smem);
  double *part = d + ((n + 1) & ~1);
  double *cache = part + OP_WARPS * 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hl = lane & 15, hf = lane >> 4;
  const int r0 = blockIdx.x * R;
  const int nr = max(0, min(R, n - r0));
  const bool rok = 2 * hl < nr;
  const int creg = min(n, 2 * OP_WARPS * K2);
  const int cs0 = creg, cg0 = min(n, creg + Cs);
  const int c_off = 2 * warp + hf;
  const int nb = gridDim.x;
  // LL layout: [2 parities][n values + nb maxima][2 words]
  const size_t stride = (size_t)(n + nb) * 2;
  double2 treg[K2];
#pragma unroll
  for (int k = 0; k < K2; ++k) {
    const int c = c_off + 2 * OP_WARPS * k;
    treg[k] = (rok && c < creg) ? *reinterpret_cast<const double2 *>(Tcm + (size_t)c * n + r0 + 2 * hl)
                                : make_double2(0.0, 0.0);
  }
  for (int i = tid; i < (cg0 - cs0) * R; i += OP_THREADS) {
    const int c = cs0 + i / R, r = i - (i / R) * R;
    cache[i] = r < nr ? Tcm[(size_t)c * n + r0 + r] : 0.0;
  }
  if (tid == 0) bad_s = 0;
  if (a.st->done) return;
  double own = 0.0;                                     // this lane's row of the last density
  if (tid < nr) own = __ldcg(((a.first_idx & 1) ? A : B) + r0 + tid);
  for (int idx = a.first_idx; idx < a.max_iter; ++idx) {
    const double *in = (idx & 1) ? A : B;
    double *out = (idx & 1) ? B : A;
    const unsigned int ep_in = ebase + idx - 1;             // epoch of the previous op sweep
    const unsigned long long *llin = ll + (size_t)((idx - 1) & 1) * stride;
    unsigned long long *llout = ll + (size_t)(idx & 1) * stride;
    const bool from_ll = idx > a.first_idx;
    for (int q0 = 0; q0 < n; q0 += OP_THREADS * 8) {
      double vi[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        vi[u] = (!from_ll && p < n) ? __ldcg(in + p) : 0.0;
      }
      if (from_ll) {
        unsigned int pending = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (q0 + tid + u * OP_THREADS < n) pending |= 1u << u;
        for (int it = 0; pending && it < (1 << 22); ++it) {
          unsigned long long w0[8], w1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int p = q0 + tid + u * OP_THREADS;
            if (pending & (1u << u))
              asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                           : "=l"(w0[u]), "=l"(w1[u]) : "l"(llin + 2 * (size_t)p) : "memory");
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if ((pending & (1u << u)) && (unsigned int)w0[u] == ep_in && (unsigned int)w1[u] == ep_in) {
              vi[u] = __longlong_as_double((long long)((w0[u] & 0xffffffff00000000ull) | (w1[u] >> 32)));
              pending &= ~(1u << u);
            }
          }
        }
        if (pending) bad_s = 1;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = q0 + tid + u * OP_THREADS;
        if (p < n) d[p] = vi[u] - __ldg(phi0 + p);
      }
    }
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const int c = c_off + 2 * OP_WARPS * k;
      if (c < creg) {
        const double dc = d[c];
        acc.x = fma(treg[k].x, dc, acc.x);
        acc.y = fma(treg[k].y, dc, acc.y);
      }
    }
    if (rok)
      for (int c = cs0 + c_off; c < cg0; c += 2 * OP_WARPS) {
        const double2 t2 = *reinterpret_cast<const double2 *>(cache + (size_t)(c - cs0) * R + 2 * hl);
        const double dc = d[c];
        acc.x = fma(t2.x, dc, acc.x);
        acc.y = fma(t2.y, dc, acc.y);
      }
    for (int c = cg0 + c_off; c < n; c += 2 * OP_WARPS * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + 2 * OP_WARPS * u;
        v[u] = (rok && cc < n) ? __ldcg(reinterpret_cast<const double2 *>(Tcm + (size_t)cc * n + r0 + 2 * hl))
                               : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + 2 * OP_WARPS * u;
        if (cc < n) {
          const double dc = d[cc];
          acc.x = fma(v[u].x, dc, acc.x);
          acc.y = fma(v[u].y, dc, acc.y);
        }
      }
    }
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 16);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 16);
    if (hf == 0) {
      part[warp * 32 + 2 * hl] = acc.x;
      part[warp * 32 + 2 * hl + 1] = acc.y;
    }
    __syncthreads();
    const unsigned int ep = ebase + idx;
    if (warp == 0) {
      double mag = 0.0;
      if (tid < nr) {
        const int q = r0 + tid;
        double s2 = part[tid];
        for (int w = 1; w < OP_WARPS; ++w) s2 += part[w * 32 + tid];
        const double trace = trace1[q] + s2;
        const double upd = (g[q] - trace) * a.gamma;
        const double nv = own + upd;
        own = nv;
        out[q] = nv;
        ll_put(llout + 2 * (size_t)q, nv, ep);
        mag = fabs(upd);
      }
      mag = warp_nanmax(mag);
      if (lane == 0) ll_put(llout + 2 * (size_t)(n + blockIdx.x), mag, ep);
    }
    // the sweep's max over all CTAs (polled; no barrier)
    double mx = 0.0;
    for (int b = tid; b < nb; b += OP_THREADS) {
      double v;
      if (!ll_get(llout + 2 * (size_t)(n + b), ep, v)) bad_s = 1;
      mx = nanmax(mx, v);
    }
    mx = warp_nanmax(mx);
    if (lane == 0) res_w[warp] = mx;
    __syncthreads();
    double res = res_w[0];
    for (int w = 1; w < OP_WARPS; ++w) res = nanmax(res, res_w[w]);
    if (bad_s) res = __longlong_as_double(0x7ff8000000000000ll);   // timeout: NaN stops the solve
    const bool conv = res <= a.tol;
    const bool last = conv || idx + 1 >= a.max_iter || bad_s;
    if (blockIdx.x == 0 && tid == 0) {
      a.history[idx] = res;
      a.st->iters = idx + 1;
      a.st->last_res = res;
      if (conv) a.st->done = 1;
      else if (idx + 1 >= a.max_iter || bad_s) a.st->done = 2;
    }
    if (last) break;
    __syncthreads();                                    // res_w / d reuse
  }
}

struct Run {
  const char *name;
  const void *fn;
  int k2;
  bool v;
  int ring_bytes;
};

int main(int argc, char **argv) {
  int sms, optin;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  Run runs[] = {
      {"product K2=12 U=8", (const void *)op_solve_pair_kernel<12>, 12, false, 0},
      {"v K2=12 U=8 bar", (const void *)op_pair_v<12, 8, false, true>, 12, true, 0},
      {"product K2=13", (const void *)op_solve_pair_kernel<13>, 13, false, 0},
      {"product K2=14", (const void *)op_solve_pair_kernel<14>, 14, false, 0},
  };
  for (auto &r : runs) cudaFuncSetAttribute(r.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
  unsigned int *ctr;
  cudaMalloc(&ctr, 4);
  unsigned long long *llbuf;
  cudaMalloc(&llbuf, 2 * (8192 + 256) * 16);
  cudaMemset(llbuf, 0, 2 * (8192 + 256) * 16);
  for (int ai = 1; ai < argc; ++ai) {
    const int n = atoi(argv[ai]);
    const int sweeps = 40;
    std::vector<double> hT((size_t)n * n), hv(n);
    srand(1);
    for (auto &x : hT) x = (rand() / (double)RAND_MAX - 0.5) * (1.0 / n);
    for (auto &x : hv) x = rand() / (double)RAND_MAX;
    double *T, *A, *B, *phi0, *tr1, *g, *hist;
    RichState *st;
    unsigned long long *slots;
    cudaMalloc(&T, hT.size() * 8);
    cudaMalloc(&A, n * 8); cudaMalloc(&B, n * 8); cudaMalloc(&phi0, n * 8);
    cudaMalloc(&tr1, n * 8); cudaMalloc(&g, n * 8); cudaMalloc(&hist, 1024 * 8);
    cudaMalloc(&st, sizeof(RichState)); cudaMalloc(&slots, 64);
    cudaMemcpy(T, hT.data(), hT.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(phi0, hv.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(tr1, hv.data(), n * 8, cudaMemcpyHostToDevice);
    for (auto &x : hv) x = 1.0 - x;
    cudaMemcpy(g, hv.data(), n * 8, cudaMemcpyHostToDevice);
    int rows = (n + sms - 1) / sms;
    rows += rows & 1;
    const int grid = (n + rows - 1) / rows;
    for (auto &r : runs) {
      const size_t fixed = op_smem_fixed<double>(n) + (r.ring_bytes > 0 ? r.ring_bytes : 0);
      const size_t avail = (size_t)(optin - 1024) - fixed;
      const int creg = std::min(n, 2 * OP_WARPS * r.k2);
      size_t cs = avail / ((size_t)rows * 8);
      if (cs > (size_t)(n - creg)) cs = n - creg;
      const size_t smem = fixed + cs * rows * 8;
      OpSolveArgs a;
      a.n = n; a.first_idx = 1; a.max_iter = sweeps + 1; a.gamma = 0.8; a.tol = -1.0;
      a.st = st; a.history = hist; a.slots = slots; a.bar = ctr; a.rows = rows; a.smem_cols = (int)cs;
      unsigned int ebase = 1000u * (unsigned)(&r - runs) + 7u;
      void *args_ll[] = {&a, &T, &A, &B, &phi0, &tr1, &g, &llbuf, &ebase};
      void *args_v[] = {&a, &T, &A, &B, &phi0, &tr1, &g, &ctr};
      void **args = r.ring_bytes < 0 ? args_ll : args_v;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemcpy(A, hv.data(), n * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(B, hv.data(), n * 8, cudaMemcpyHostToDevice);
        cudaMemset(st, 0, sizeof(RichState));
        cudaMemset(slots, 0, 64);
        cudaMemset(ctr, 0, 4);
        ebase += 100;
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(r.fn, dim3(grid), dim3(OP_THREADS), args, smem, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      cudaError_t err = cudaGetLastError();
      std::vector<double> out(n);
      cudaMemcpy(out.data(), (sweeps & 1) ? A : B, n * 8, cudaMemcpyDeviceToHost);
      double cs_ = 0;
      for (double x : out) cs_ += x;
      RichState hs;
      cudaMemcpy(&hs, st, sizeof hs, cudaMemcpyDeviceToHost);
      printf("%-24s n=%d rows=%d grid=%d smem_cols=%zu streamed=%d: %.2f us/sweep (iters %d) sum %.17g %s\n",
             r.name, n, rows, grid, cs, (int)(n - creg - cs), best * 1000 / sweeps, hs.iters, cs_,
             cudaGetErrorString(err));
    }
    cudaFree(T); cudaFree(A); cudaFree(B); cudaFree(phi0); cudaFree(tr1); cudaFree(g);
    cudaFree(hist); cudaFree(st); cudaFree(slots);
  }
}
