// Box-solve arguments and the sparse right-hand-side corrections shared by
// the register-engine kernels (box_reg.cuh) and the corrections() API.
#pragma once

#include "common.cuh"

namespace kfbi {

struct BoxArgs {
  int m, logm;
  const double *lam;      // [m+1] (2cos(p pi/m) - 2)/h^2 at p = 1..m-1
  double kre, kim;        // kappa
  double inv4m2;          // 1 / (4 m^2), exact power of two
  double h2;              // h^2 (tridiagonal column pass, box_tri.cuh)
  // cyclic-reduction (FACR) form of the box solve, box_tri.cuh / box_facr.cuh:
  int red;                // column stage on the even-row system (root r^2)
  int trow;               // recurrence along x of one grid row (odd rows)
  int row_step;           // grid rows per slab row of the inverse row pass (1, or 2)
  double tb_re, tb_im;    // trow: beta - 1 of the x recurrence (1 + kappa h^2 / 2)
  double tscale;          // trow: output scale (1)
  void *gsum;             // scratch for the group sums (n_groups slots of 16 bytes)
  const int2 *oc_list;    // FACR: solve only these (odd row, 16-chunk) pieces of the odd rows
  int n_oc;               // (trace-only first sweep; nullptr: every odd row)
  const int2 *span;       // FACR: per odd row (j - 1) / 2, the chunk range [x, y] the caller
                          // reads (x > y: none); nullptr: whole rows
  const unsigned char *row_need;  // FACR inverse pass: per even row j / 2, 0 = nobody reads it
  unsigned char *rowz;    // FACR: per reduced row, 1 = its forward output is zero (written by the
                          // forward pass, which then skips the panel stores; read by the columns)
  unsigned char *zbuf;    // the plan's flag buffer (the FACR launcher sets rowz = zbuf)
  void *panels;
  const int *done;        // early-exit flag (Richardson sweeps), may be null
  const double2 *twg;     // [m] exp(-2 pi i q / m)        (register engine)
  const double *sinv;     // [m] sin(pi j / m)              (register engine)
  // Row slabs (one GPU: a single slab, rows = m, row0 = 0, npl = all panels).
  // This rank's row pass covers grid rows [row0, row0 + rows); its field
  // arrays hold exactly those rows (row j at (j - row0) * (m + 1)), and its
  // panel buffer is [panel][rows][w].  Its column pass covers panels
  // [pp0, pp0 + npl) of every row, received as nranks blocks [rank][npl][rows][w].
  int rows, row0, pp0, npl;
  int ring_end;           // the field array also holds row m (zero ring)
  // Transposes fused into the stores (slab_*_p2p): when dst[0] != null the
  // forward row pass writes each panel chunk straight into the column-pass
  // buffer of the panel's owner, and the column pass writes each row chunk
  // into the row-pass buffer of the row's owner (peer device memory over
  // NVLink, or other buffers of the same device); no all-to-all follows.
  int nranks, rank;
  void *dst[8];
};

// Destination of panel-row element (panel pp, slab row r, half w) written by
// the forward row pass: own buffer [pp][R] or the owner's [rank][pl][R].
KFBI_DEV double2 *rows_fwd_dst(const BoxArgs &a, int pp, int r, int w) {
  if (!a.dst[0]) return static_cast<double2 *>(a.panels) + ((size_t)pp * a.rows + r) * 2 + w;
  const int h = pp / a.npl, pl = pp - h * a.npl;
  return static_cast<double2 *>(a.dst[h]) + (((size_t)a.rank * a.npl + pl) * a.rows + r) * 2 + w;
}

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
  const T *cval = nullptr;  // precomputed group sums (the FACR passes), or null
};

// Correction at one irregular node: sum over its arm records, in record
// order, of sigma * (j_u + j_1 d + 0.5 j_2 d^2) (interface.py:228-237).
template <typename T>
KFBI_DEV T group_correction(const CorrArgs<T> &c, int g) {
  using S = Sc<T>;
  if (c.cval) return c.cval[g];
  const int r0 = c.group_start[g], r1 = c.group_start[g + 1];
  T acc = S::zero();
  if (r1 - r0 <= 4) {
    // a node has at most four crossing edges: every gather in flight at once,
    // then the same ordered sum as the loop below
    const int cnt = r1 - r0;
    int e[4];
    double d[4], sg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e[k] = k < cnt ? c.rec_edge[r0 + k] : 0;
      d[k] = k < cnt ? c.rec_d[r0 + k] : 0.0;
      sg[k] = k < cnt ? c.rec_sigma[r0 + k] : 0.0;
    }
    T j0[4], j1[4], j2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      j0[k] = k < cnt ? c.jv[3 * e[k]] : S::zero();
      j1[k] = k < cnt ? c.jv[3 * e[k] + 1] : S::zero();
      j2[k] = k < cnt ? c.jv[3 * e[k] + 2] : S::zero();
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < cnt) {
        T v = S::add(S::add(j0[k], S::rmul(j1[k], d[k])), S::rmul(S::rmul(j2[k], 0.5), d[k] * d[k]));
        v = S::rmul(v, sg[k]);
        acc = k == 0 ? v : S::add(acc, v);
      }
    }
    return acc;
  }
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

// The group sums into a compact array (the FACR passes read each one once
// instead of re-walking the records in every thread that needs it).
template <typename T>
__global__ void __launch_bounds__(256) group_sums_kernel(CorrArgs<T> c, int m, T *out) {
  const int n_groups = c.row_group[m + 1];
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n_groups; g += gridDim.x * blockDim.x)
    out[g] = group_correction<T>(c, g);
}

// Dense scatter of the group sums (the standalone corrections() API).
template <typename T>
__global__ void scatter_groups_kernel(CorrArgs<T> c, int n_groups, T *out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n_groups) out[c.group_node[g]] = group_correction<T>(c, g);
}

}  // namespace kfbi

#ifdef KFBI_MAIN_TU   // one definition (a plain __global__) in the main unit
// ---------------------------------------------------------------------------
// Peer-flag barrier between the fused slab passes (kfbi_p2p_barrier): rank r
// publishes `epoch` into slot r of every rank's flag array (system-scope
// release over NVLink), then waits until every slot of its own array holds
// at least `epoch` (acquire).  One warp; lane h talks to rank h.  The spin is
// bounded (max_spins polls): a missing peer sets *timed_out instead of hanging.
struct P2pFlags {
  unsigned long long *flags[8];
};

__global__ void p2p_barrier_kernel(P2pFlags f, int nranks, int rank, unsigned long long epoch,
                                   long long max_spins, int *timed_out) {
  const int h = threadIdx.x;
  if (h >= nranks) return;
  __threadfence_system();
  unsigned long long *slot = f.flags[h] + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
  const unsigned long long *mine = f.flags[rank] + h;
  for (long long it = 0;; ++it) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    if (it >= max_spins) {
      if (timed_out) atomicExch(timed_out, 1);
      break;
    }
    __nanosleep(64);
  }
  __threadfence_system();
}
#endif  // KFBI_MAIN_TU
