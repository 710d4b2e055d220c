// C ABI of the B200-native KFBI hot path (include/kfbi_b200.h).
//
// One translation unit: the device kernels live in the *.cuh headers, this
// file owns the plan object (device tables + scratch), launch bookkeeping,
// per-kernel-name CUDA-event timing (the Backend.timings contract of
// engine.py:84-95) and error reporting.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#define KFBI_MAIN_TU
#include "host_common.h"
#include "interface_kernels.cuh"
#include "gmres.cuh"
#include "classify.cuh"
#include "box_tri.cuh"
#include "stepping_kernels.cuh"

using namespace kfbi;

namespace {

thread_local std::string g_last_error;

kfbi_status fail(kfbi_status code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

const char *kKernelNames[KFBI_N_KERNEL_NAMES] = {
    "classify-nodes", "edge-intersections", "jumps-and-corrections",
    "transform-rows", "transform-cols",     "diagonal-scale",
    "extract-traces", "density-update",     "rhs-update"};

// NVTX ranges (nsys / ncu --nvtx) carry the reference's kernel names
const char *kNvtxNames[KFBI_N_KERNEL_NAMES] = {
    "kfbi:classify-nodes", "kfbi:edge-intersections", "kfbi:jumps-and-corrections",
    "kfbi:transform-rows", "kfbi:transform-cols",     "kfbi:diagonal-scale",
    "kfbi:extract-traces", "kfbi:density-update",     "kfbi:rhs-update"};

struct Pending {
  int name;
  cudaEvent_t a, b;
};

template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t count) {
    if (count <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    // defined contents from the start (state structs are copied to the host
    // whole, padding included; compute-sanitizer initcheck clean)
    if (e == cudaSuccess) e = cudaMemset(p, 0, count * sizeof(T));
    if (e == cudaSuccess) n = count;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
cudaError_t upload(DevBuf<T> &b, const T *host, size_t count) {
  cudaError_t e = b.ensure(count ? count : 1);
  if (e != cudaSuccess) return e;
  if (count) e = cudaMemcpy(b.p, host, count * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

struct kfbi_plan {
  int device = 0;
  int m = 0, logm = 0;
  double h = 0.0;
  DevBuf<double> lam;
  DevBuf<double2> panels;       // m*m complex slots (sized for c128)
  DevBuf<double2> twg;          // register engine: exp(-2 pi i q / m), q < m
  DevBuf<double> sinv;          // register engine: sin(pi j / m), j < m
  // geometry
  bool has_geo = false;
  int n_ctl = 0, n_edges = 0, n_rec = 0, n_groups = 0, w_ld = 0;
  DevBuf<double> W;
  // edge values: W rows (streamed) or the matrix-free spectral form
  int interp_mode = 0;              // 0 auto, 1 W rows, 2 spectral
  int col_mode = 0;                 // 0 auto, 1 tridiagonal recurrences, 2 DST-I engine
  bool spec_ok = false;             // equispaced controls, even n >= 32
  bool w_ready = false;             // W built / uploaded
  bool w_explicit = false;          // W given by the caller (cubic rows)
  DevBuf<double> edge_theta_d, ctl_theta_d;
  DevBuf<double2> spec, spec_part;
  DevBuf<int> edge_perm;            // edges grouped by axis, 4 per group, -1 pads
  int n_perm = 0;
  DevBuf<unsigned int> spec_ctr;    // per frequency block, self-resetting
  DevBuf<signed char> edge_axis;
  DevBuf<int> rec_edge, group_start, group_node, row_group, stencil;
  DevBuf<double> rec_d, rec_sigma, deriv_col, speed, tangent, normal, dtan_ds, inv3;
  DevBuf<double> ainv_rows, jcoef;
  // OneSidedExtractor tables (Neumann BVPs)
  bool has_os = false;
  DevBuf<int> os_stencil;
  DevBuf<double> os_rows;
  DevBuf<unsigned char> os_fb;
  // per-sweep scratch (sized for c128)
  DevBuf<double2> d1, psi_s, jm, jv;
  DevBuf<double> history;
  DevBuf<RichState> st;
  // operator form (trace operator T of one kappa / dtype)
  DevBuf<double2> Top, phi0, phi_prev, trace1, trace_tmp, zvec, evec, out3, ufield;
  DevBuf<double2> phik1;
  // GMRES (gmres.cuh) scratch
  DevBuf<double2> gm_V, gm_w, gm_H, gm_sn, gm_g, gm_y, gm_part, gm_tr;
  DevBuf<double> gm_cs, gm_np;
  DevBuf<GmresState> gm_st;
  // stencil nodes grouped by grid row (trace-only sweep 1 of the operator form)
  DevBuf<int> sn_rows, sn_rowptr, sn_cols, sn_map;
  DevBuf<int2> oc_list;             // (odd row, 16-element chunk) pairs holding stencil nodes
  DevBuf<int2> fc_span;             // kfbi_plan_set_field_chunks: per odd row, the chunk range read
  int n_fc = 0;
  DevBuf<unsigned char> need_trace, need_field;   // per even row j / 2: read by a trace sweep / a masked field
  DevBuf<unsigned char> rowz;                     // FACR zero-row flags (per reduced row)
  double frac[4] = {1.0, 1.0, 1.0, 1.0};         // kfbi_plan_work_fractions
  int n_oc = 0;                     // 0: the sparse odd-row pass does not apply
  bool facr_trace = true;           // env KFBI_FACR_TRACE=0: sweep 1 forms the whole field
  DevBuf<double2> gsum;             // group sums of the FACR passes
  int sn_nrows = 0, sn_nodes = 0;
  bool trace_sweep = false;         // kfbi_plan_set_trace_sweep (opt-in: measured no gain)
  bool facr = true;                 // kfbi_plan_set_facr: cyclic-reduction box solve
  bool edges_smem = true;           // W-row edge values with JM staged per CTA (env KFBI_EDGES_SMEM=0: per warp)
  bool op_cta = true;               // operator sweeps of n_ctl <= 160 in one CTA (env KFBI_OP_CTA=0: grid kernels)
  bool edges_full = true;           // staged edge values with all of JM in shared memory (env KFBI_EDGES_FULL=0)
  bool ext_zero = false;            // kfbi_plan_set_exterior_zero: masked outputs already zero outside the mask
  const int *int_idx = nullptr;     // kfbi_plan_set_interior_list: the mask's interior nodes (caller-owned)
  int64_t n_int = 0;
  DevBuf<double2> sn_vals, sn_v13;
  DevBuf<int> skip;
  DevBuf<StepLog> log;
  int log_cap = 0;
  bool op_valid = false;
  int op_dtype = -1;
  int op_bc = -1;                   // bc_kind the operator was built for
  double op_kre = 0.0, op_kim = 0.0;
  DevBuf<unsigned long long> red;   // reduction slots
  RichState *st_host = nullptr;     // pinned mirror
  unsigned long long *red_host = nullptr;
  // timing / accounting
  bool timing = true;
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  double ms[KFBI_N_KERNEL_NAMES] = {0};
  int64_t calls[KFBI_N_KERNEL_NAMES] = {0};
  int64_t launches = 0;

  cudaEvent_t take_event() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

kfbi_status kfbi_fail(kfbi_status code, const std::string &msg) { return fail(code, msg); }

KfbiLaunchTok kfbi_launch_begin(kfbi_plan *p, int name, cudaStream_t s) {
  KfbiLaunchTok t;
  nvtxRangePushA(kNvtxNames[name]);
  if (p->timing) {
    t.a = p->take_event();
    t.b = p->take_event();
    cudaEventRecord(t.a, s);
  }
  return t;
}

kfbi_status kfbi_launch_end(kfbi_plan *p, int name, cudaStream_t s, KfbiLaunchTok t, cudaError_t e) {
  nvtxRangePop();
  cudaError_t e2 = cudaGetLastError();
  if (e == cudaSuccess) e = e2;
  if (p->timing) {
    cudaEventRecord(t.b, s);
    p->pending.push_back(Pending{name, t.a, t.b});
  }
  p->calls[name] += 1;
  p->launches += 1;
  if (e != cudaSuccess)
    return fail(KFBI_E_CUDA, std::string("kernel '") + kKernelNames[name] +
                                 "': launch failed: " + cudaGetErrorString(e));
  return KFBI_OK;
}

namespace {

template <typename F>
kfbi_status launch(kfbi_plan *p, int name, cudaStream_t s, F &&fn) {
  return kfbi_launch(p, name, s, static_cast<F &&>(fn));
}

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

kfbi_status check_plan(kfbi_plan *p) {
  if (!p) return fail(KFBI_E_CONFIG, "null plan");
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return KFBI_OK;
}

kfbi_status check_geo(kfbi_plan *p) {
  KFBI_TRY(check_plan(p));
  if (!p->has_geo) return fail(KFBI_E_CONFIG, "plan has no geometry (call kfbi_plan_set_geometry)");
  return KFBI_OK;
}

BoxArgs box_args(kfbi_plan *p, double kre, double kim, const int *done) {
  BoxArgs a;
  a.m = p->m;
  a.logm = p->logm;
  a.lam = p->lam.p;
  a.kre = kre;
  a.kim = kim;
  a.inv4m2 = 1.0 / (4.0 * (double)p->m * (double)p->m);
  a.h2 = p->h * p->h;
  a.red = 0;
  a.trow = 0;
  a.row_step = 1;
  a.tb_re = a.tb_im = 0.0;
  a.tscale = 1.0;
  a.gsum = p->gsum.p;
  a.panels = p->panels.p;
  a.done = done;
  a.twg = p->twg.p;
  a.sinv = p->sinv.p;
  a.rows = p->m;             // one slab: the whole grid
  a.row0 = 0;
  a.pp0 = 0;
  a.npl = 0;                 // set per dtype by the launcher
  a.ring_end = 1;
  a.nranks = 1;
  a.rank = 0;
  for (int h = 0; h < 8; ++h) a.dst[h] = nullptr;
  a.oc_list = nullptr;
  a.n_oc = 0;
  a.span = nullptr;
  a.row_need = nullptr;
  a.rowz = nullptr;          // set by the FACR launcher only
  a.zbuf = p->rowz.p;
  return a;
}

// Slab geometry of rank `rank` of `nranks` (rows and panels split evenly).
kfbi_status slab_args(kfbi_plan *p, bool cplx, int nranks, int rank, BoxArgs &a) {
  const int m = p->m;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks & (nranks - 1)) != 0)
    return fail(KFBI_E_CONFIG, "slab: nranks must be a power of two and 0 <= rank < nranks");
  const int npanels = cplx ? m / 2 : m / 4;
  if (m / nranks < 2 || npanels % nranks != 0)
    return fail(KFBI_E_CONFIG, "slab: too many ranks for this grid");
  a.rows = m / nranks;
  a.row0 = rank * a.rows;
  a.npl = npanels / nranks;
  a.pp0 = rank * a.npl;
  a.ring_end = 0;
  a.nranks = nranks;
  a.rank = rank;
  return KFBI_OK;
}

template <typename T>
CorrArgs<T> corr_args(kfbi_plan *p, const T *jv) {
  CorrArgs<T> c;
  c.jv = jv;
  c.row_group = p->row_group.p;
  c.group_start = p->group_start.p;
  c.group_node = p->group_node.p;
  c.rec_edge = p->rec_edge.p;
  c.rec_d = p->rec_d.p;
  c.rec_sigma = p->rec_sigma.p;
  return c;
}

CtlGeom ctl_geom(kfbi_plan *p) {
  CtlGeom g;
  g.n = p->n_ctl;
  g.deriv_col = p->deriv_col.p;
  g.speed = p->speed.p;
  g.tangent = p->tangent.p;
  g.normal = p->normal.p;
  g.dtan_ds = p->dtan_ds.p;
  g.inv3 = p->inv3.p;
  return g;
}

ExtractArgs extract_args(kfbi_plan *p, bool onesided = false) {
  ExtractArgs x;
  x.n = p->n_ctl;
  x.m = p->m;
  x.h = p->h;
  x.inv_h = 1.0 / p->h;
  x.stencil = p->stencil.p;
  x.ainv_rows = p->ainv_rows.p;
  x.jcoef = p->jcoef.p;
  x.normal = p->normal.p;
  x.os_stencil = onesided ? p->os_stencil.p : nullptr;
  x.os_rows = onesided ? p->os_rows.p : nullptr;
  x.os_fb = onesided ? p->os_fb.p : nullptr;
  return x;
}

// Column stage choice (kfbi_plan_set_colsolver).  The reference divides by
// lam_p + lam_q - kappa with lam_q = (2 cos(q pi / M) - 2) / h^2 rounded in
// fp64 (boxsolve.py:38-44): its low-mode eigenvalues carry absolute errors up
// to ~4.4e-16 / h^2, i.e. the reference applies the exact discrete inverse
// only up to E = (4.4e-16 / h^2) / min |lam_p + lam_q - kappa| relative.  The
// tridiagonal recurrences apply the exact three-point inverse, so they agree
// with the reference to ~E; auto mode uses them when E <= 1e-11 (every
// time-stepping kappa: 2c/tau, 1/(theta tau^2), 2i/tau) and the DST-I engine,
// which shares the reference's eigenvalue table, otherwise (kappa ~ 0).
double col_deviation_bound(const kfbi_plan *p, double kre, double kim) {
  if (kre < 0.0) return 1.0;                  // sums may approach kappa: no bound
  const double h2 = p->h * p->h;
  const double lam1 = (2.0 * std::cos(M_PI / p->m) - 2.0) / h2;
  const double dre = 2.0 * lam1 - kre;        // the smallest |lam_p + lam_q - kappa|
  const double dmin = std::sqrt(dre * dre + kim * kim);
  return (4.4e-16 / h2) / dmin;
}

bool col_use_tri(const kfbi_plan *p, double kre, double kim) {
  if (p->col_mode == 1) return true;
  if (p->col_mode == 2) return false;
  return col_deviation_bound(p, kre, kim) <= 1e-11;
}

template <bool CPLX>
kfbi_status box_passes_reg(kfbi_plan *p, const BoxArgs &a, const void *rhs, double sign,
                           const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                           void *u, cudaStream_t s, int passes = 7) {
  const bool tri = col_use_tri(p, a.kre, a.kim);
  // one level of cyclic reduction (box_facr.cuh): half the row transforms;
  // single slab, full solve, tridiagonal-eligible kappa, 64 <= M <= 8192
  if (passes == 7 && tri && p->facr && a.nranks == 1 && !a.dst[0] && a.rows == p->m && p->m >= 64 &&
      (p->m <= 8192 || (!CPLX && p->m == 16384)))
    passes = 8;
  if constexpr (CPLX) return box_dirichlet_c128(p, p->logm, tri, a, rhs, sign, c, u, s, passes);
  else return box_dirichlet_f64(p, p->logm, tri, a, rhs, sign, c, u, s, passes);
}

// The three passes of one box solve.  rhs is an (M+1)^2 field (scaled by
// sign); jv != nullptr fuses the jump corrections of the plan's geometry.
template <bool CPLX>
kfbi_status box_passes(kfbi_plan *p, double kre, double kim, const void *rhs, double sign,
                       const void *jv, void *u, const int *done, cudaStream_t s) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  BoxArgs a = box_args(p, kre, kim, done);
  a.npl = CPLX ? p->m / 2 : p->m / 4;
  CorrArgs<T> c = corr_args<T>(p, static_cast<const T *>(jv));
  if (!jv) c.jv = nullptr;
  return box_passes_reg<CPLX>(p, a, rhs, sign, c, u, s);
}

// One pass of the slab-decomposed box solve (kfbi_slab_*).
// peers != nullptr: the pass stores its output straight into peers[h], the
// buffer of rank h (the all-to-all fused into the stores).
kfbi_status slab_pass(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, int passes, double kre,
                      double kim, const void *rhs, double sign, const void *jv, void *panels,
                      void *u, void *stream, void *const *peers = nullptr) {
  KFBI_TRY(check_plan(p));
  if (!sl || (!panels && !(passes == 1 && peers))) return fail(KFBI_E_CONFIG, "slab: null argument");
  const bool cplx = dtype == KFBI_C128;
  if (!cplx && kim != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  if (jv && !p->has_geo) return fail(KFBI_E_CONFIG, "slab: corrections need the plan's geometry");
  BoxArgs a = box_args(p, kre, kim, nullptr);
  KFBI_TRY(slab_args(p, cplx, sl->nranks, sl->rank, a));
  a.panels = panels;
  if (peers) {
    if (sl->nranks > KFBI_MAX_PEERS) return fail(KFBI_E_CONFIG, "slab p2p: at most 8 ranks");
    for (int h = 0; h < sl->nranks; ++h) {
      if (!peers[h]) return fail(KFBI_E_CONFIG, "slab p2p: null peer buffer");
      a.dst[h] = peers[h];
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (cplx) {
    CorrArgs<double2> c = corr_args<double2>(p, static_cast<const double2 *>(jv));
    if (!jv) c.jv = nullptr;
    return box_passes_reg<true>(p, a, rhs, sign, c, u, s, passes);
  }
  CorrArgs<double> c = corr_args<double>(p, static_cast<const double *>(jv));
  if (!jv) c.jv = nullptr;
  return box_passes_reg<false>(p, a, rhs, sign, c, u, s, passes);
}

// neumann-zero closure: DCT-I passes (box_neu.cuh, box_neu_*.cu), one GPU
template <bool CPLX>
kfbi_status box_neu_passes(kfbi_plan *p, double kre, double kim, const void *rhs, double sign,
                           const void *jv, void *u, const int *done, cudaStream_t s) {
  using T = typename std::conditional<CPLX, double2, double>::type;
  if (kre == 0.0 && kim == 0.0)
    return fail(KFBI_E_CONFIG, "neumann-zero box with kappa = 0 is singular (constant null mode)");
  BoxArgs a = box_args(p, kre, kim, done);
  CorrArgs<T> c = corr_args<T>(p, static_cast<const T *>(jv));
  if (!jv) c.jv = nullptr;
  if constexpr (CPLX) return box_neumann_c128(p, p->logm, a, rhs, sign, c, u, s);
  else return box_neumann_f64(p, p->logm, a, rhs, sign, c, u, s);
}

kfbi_status box_dispatch(kfbi_plan *p, int dtype, double kre, double kim, const void *rhs,
                         double sign, const void *jv, void *u, const int *done,
                         cudaStream_t s, int box_bc = KFBI_DIRICHLET_ZERO) {
  if (dtype != KFBI_C128 && kim != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  if (box_bc == KFBI_NEUMANN_ZERO) {
    if (dtype == KFBI_C128) return box_neu_passes<true>(p, kre, kim, rhs, sign, jv, u, done, s);
    return box_neu_passes<false>(p, kre, kim, rhs, sign, jv, u, done, s);
  }
  if (box_bc != KFBI_DIRICHLET_ZERO) return fail(KFBI_E_CONFIG, "unknown box boundary condition");
  if (dtype == KFBI_C128) return box_passes<true>(p, kre, kim, rhs, sign, jv, u, done, s);
  return box_passes<false>(p, kre, kim, rhs, sign, jv, u, done, s);
}

// jumps (two kernels) for dtype T; jm is SoA [6][n].
template <typename T>
kfbi_status jumps_T(kfbi_plan *p, double kre, double kim, const void *phi, const void *psi,
                    const void *fg, double fg_sign, void *jm, const int *done, cudaStream_t s) {
  CtlGeom g = ctl_geom(p);
  const int warps_per_block = 8;
  const int blocks = (p->n_ctl + warps_per_block - 1) / warps_per_block;
  T *d1 = reinterpret_cast<T *>(p->d1.p);
  T *ps = reinterpret_cast<T *>(p->psi_s.p);
  const T *ph = static_cast<const T *>(phi);
  const T *pv = static_cast<const T *>(psi);
  // shared-memory circulant kernels when both vectors and D fit (n_ctl up to
  // ~5,000); the warp-per-output kernels otherwise (C5)
  static int optin = 0;
  static bool attr = false;
  if (!attr) {
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    KFBI_CUDA(cudaFuncSetAttribute(circ_block_kernel<T, 2, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "jumps-and-corrections");
    KFBI_CUDA(cudaFuncSetAttribute(circ_block_kernel<T, 1, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "jumps-and-corrections");
    KFBI_CUDA(cudaFuncSetAttribute(circ_block_kernel<T, 1, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "jumps-and-corrections");
    attr = true;
  }
  const int n = p->n_ctl;
  if (circ_smem_bytes<T>(n, 2) <= (size_t)optin) {
    const int cb = (n + CIRC_OUT - 1) / CIRC_OUT;
    JumpArgs<T> ja{ph, pv, d1, ps, static_cast<const T *>(fg), fg_sign, kre, kim, static_cast<T *>(jm)};
    if (ph && pv) {
      KFBI_TRY(launch(p, KFBI_K_JUMPS, s, [&] {
        circ_block_kernel<T, 2, false><<<cb, 256, circ_smem_bytes<T>(n, 2), s>>>(g, ph, pv, d1, ps, ja, done);
      }));
    } else if (ph || pv) {
      KFBI_TRY(launch(p, KFBI_K_JUMPS, s, [&] {
        circ_block_kernel<T, 1, false><<<cb, 256, circ_smem_bytes<T>(n, 1), s>>>(
            g, ph ? ph : pv, nullptr, ph ? d1 : ps, nullptr, ja, done);
      }));
    }
    return launch(p, KFBI_K_JUMPS, s, [&] {
      circ_block_kernel<T, 1, true><<<cb, 256, circ_smem_bytes<T>(n, 1), s>>>(
          g, ph ? d1 : nullptr, nullptr, nullptr, nullptr, ja, done);
    });
  }
  KFBI_TRY(launch(p, KFBI_K_JUMPS, s, [&] {
    jumps_d1_kernel<T><<<blocks, 32 * warps_per_block, 0, s>>>(g, ph, pv, d1, ps, done);
  }));
  KFBI_TRY(launch(p, KFBI_K_JUMPS, s, [&] {
    jumps_d2_kernel<T><<<blocks, 32 * warps_per_block, 0, s>>>(
        g, ph, pv, d1, ps, static_cast<const T *>(fg), fg_sign, kre, kim,
        static_cast<T *>(jm), done);
  }));
  return KFBI_OK;
}

// W rows built on the device from the crossing and control parameters
// (interp_rows trig branch) when first needed: the W-row path of edges_T,
// kfbi_plan_copy_w.  The spectral path never builds them.
kfbi_status ensure_w(kfbi_plan *p) {
  if (p->w_ready) return KFBI_OK;
  if (!p->edge_theta_d.p || !p->ctl_theta_d.p) return fail(KFBI_E_CONFIG, "W rows: no crossing parameters");
  cudaError_t e = p->W.ensure((size_t)p->n_edges * p->w_ld + 1);
  if (e == cudaSuccess && p->n_edges > 0) {
    w_build_kernel<<<148 * 16, 256>>>(p->n_edges, p->n_ctl, p->w_ld, p->edge_theta_d.p, p->ctl_theta_d.p,
                                      p->W.p);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("W build: ") + cudaGetErrorString(e));
  p->w_ready = true;
  return KFBI_OK;
}


// Matrix-free edge values: the spectrum of the used JM columns, then one
// k-sum per edge (interface_kernels.cuh).  The spectrum stays resident in
// shared memory when it fits (one CTA per SM); otherwise it is staged in
// chunks (C5-size n_ctl).
template <typename T>
kfbi_status edges_spectral(kfbi_plan *p, const void *jm, void *jv, const int *done, cudaStream_t s) {
  constexpr int NP = std::is_same<T, double2>::value ? 2 : 1;
  constexpr int R = SPEC_COLS * NP;
  constexpr int EB = NP == 1 ? 4 : 2;          // edges per group (perm groups of 4)
  static int sms = 0, optin = 0;
  static bool attr = false;
  if (!attr) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    KFBI_CUDA(cudaFuncSetAttribute(edges_spectral_kernel<T, EB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(R * SPEC_KC * sizeof(double2))), "jumps-and-corrections");
    KFBI_CUDA(cudaFuncSetAttribute(edges_spectral_res_kernel<T, EB>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, optin), "jumps-and-corrections");
    KFBI_CUDA(cudaFuncSetAttribute(spec_block_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   optin - 1024), "jumps-and-corrections");
    attr = true;
  }
  const int n = p->n_ctl, K = n / 2 + 1;
  const int kb = (K + 31) / 32;
  static const int y_env = [] {
    const char *e = std::getenv("KFBI_SPEC_Y");        // control splits per frequency block
    return e ? std::atoi(e) : 0;
  }();
  int Y = (2 * sms) / kb;
  Y = Y < 1 ? 1 : (Y > 8 ? 8 : Y);
  if (y_env > 0) Y = y_env;
  // the staged control range of a CTA must fit next to the reduction buffer
  const size_t red_bytes = (size_t)16 * R * 32 * sizeof(double2);
  while (((size_t)SPEC_COLS * jn_max(n, Y) * sizeof(T) + 15) + red_bytes + (size_t)R * 32 * sizeof(double2) >
             (size_t)(optin - 1024) && Y < 64)
    ++Y;
  // Y <= 8 splits run as one thread-block cluster per frequency block (the
  // partial sums meet in distributed shared memory; KFBI_SPEC_CLUSTER=0: the
  // global partials + last-CTA path)
  static const bool cl_env = [] {
    const char *v = std::getenv("KFBI_SPEC_CLUSTER");
    return !(v && v[0] == '0');
  }();
  // (only where several CTAs fit per SM: with one CTA of ~200 KB per SM, C5's
  // 8192 controls, the full bench measured 109 -> 155 ms per solve)
  const size_t spec_base = red_bytes + (((size_t)SPEC_COLS * jn_max(n, Y) * sizeof(T) + 15) & ~(size_t)15);
  const bool clustered = cl_env && Y > 1 && Y <= 8 && spec_base <= ((size_t)96 << 10);
  const size_t spec_smem = spec_base + (clustered ? (size_t)R * 32 * sizeof(double2) : 0);
  cudaError_t e = p->spec.ensure((size_t)2 * SPEC_COLS * K);
  if (e == cudaSuccess) e = p->spec_part.ensure((size_t)Y * 2 * SPEC_COLS * K);
  if (e == cudaSuccess && p->spec_ctr.n < (size_t)kb) {
    e = p->spec_ctr.ensure((size_t)kb);
    if (e == cudaSuccess) e = cudaMemset(p->spec_ctr.p, 0, (size_t)kb * sizeof(unsigned int));
  }
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("spectral edges: ") + cudaGetErrorString(e));
  if (p->n_edges == 0) return KFBI_OK;
  KFBI_TRY(launch(p, KFBI_K_JUMPS, s, [&] {
    if (!clustered) {
      spec_block_kernel<T><<<dim3(kb, Y), 512, spec_smem, s>>>(
          n, K, static_cast<const T *>(jm), p->spec_part.p, p->spec.p, p->spec_ctr.p, 0);
      return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kb, Y);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = spec_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = Y;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, spec_block_kernel<T>, n, K, static_cast<const T *>(jm), p->spec_part.p,
                              p->spec.p, p->spec_ctr.p, 1);
  }));
  const int ngroups = p->n_perm / EB;
  const size_t res_bytes = (size_t)R * K * sizeof(double2);
  if (res_bytes <= (size_t)optin) {
    return launch(p, KFBI_K_JUMPS, s, [&] {
      edges_spectral_res_kernel<T, EB><<<sms, 512, res_bytes, s>>>(
          ngroups, n, K, p->edge_perm.p, p->edge_theta_d.p, p->edge_axis.p, p->spec.p,
          static_cast<T *>(jv), done);
    });
  }
  return launch(p, KFBI_K_JUMPS, s, [&] {
    edges_spectral_kernel<T, EB><<<(ngroups + 7) / 8, 256, R * SPEC_KC * sizeof(double2), s>>>(
        ngroups, n, K, p->edge_perm.p, p->edge_theta_d.p, p->edge_axis.p, p->spec.p,
        static_cast<T *>(jv), done);
  });
}

// Auto mode: the spectral form when the W stream it replaces is large (its
// cost is fp64 work ~ n_edges n_ctl, the stream's HBM bytes 8 n_edges n_ctl;
// measured at 4096^2: spectral 59 us vs W 80 us for the 340 MB flower rows,
// 69 us vs 61 us for the 116 MB star rows), always when forced (mode 2).
#ifndef KFBI_SPEC_MIN_BYTES
#define KFBI_SPEC_MIN_BYTES (192ull << 20)
#endif
bool use_spectral(const kfbi_plan *p) {
  if (!p->spec_ok || p->w_explicit || p->interp_mode == 1) return false;
  if (p->interp_mode == 2) return true;
  return (unsigned long long)p->n_edges * p->n_ctl * 8ull >= KFBI_SPEC_MIN_BYTES;
}

template <typename T>
kfbi_status edges_T(kfbi_plan *p, const void *jm, void *jv, const int *done, cudaStream_t s) {
  if (use_spectral(p)) return edges_spectral<T>(p, jm, jv, done, s);
  KFBI_TRY(ensure_w(p));
  // one wave of 2 CTAs per SM, the edges spread evenly over its warps in
  // contiguous ranges of at most EW (a partial second wave ran on half the
  // SMs); larger problems use more waves of full ranges
  constexpr int EW = std::is_same<T, double2>::value ? 4 : 8, U = 2;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  if (p->n_edges == 0) return KFBI_OK;
  // JM staged per CTA (corr_edges_smem_kernel, one CTA of CE_WARPS warps per SM)
  // when a wave of warps covers the edges with <= 4 rows each: 61 -> 46 us for
  // the star3 c128 rows at 4096^2, 22 -> 16 us at 1024^2; with more rows per
  // warp the per-warp form's deeper load queue wins (flower f64 at 4096^2:
  // 79 vs 92 us; profiles/r2_v31_edges.log)
  const int wave_s = sms * CE_WARPS;
  const int pw_s = (p->n_edges + wave_s - 1) / wave_s;
  if (p->edges_smem && pw_s <= 4) {
    const int pw = pw_s;
    static int optin_ce = 0;
    if (!optin_ce) cudaDeviceGetAttribute(&optin_ce, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    const size_t full_bytes = (size_t)5 * 2 * ((p->n_ctl + 1) / 2) * sizeof(T);
    auto go = [&](auto ew) {
      constexpr int E = decltype(ew)::value;
      EdgeArgs ea{p->n_edges, p->n_ctl, p->w_ld, pw, p->W.p, p->edge_axis.p};
      const int warps = (p->n_edges + pw - 1) / pw;
      const int blocks = (warps + CE_WARPS - 1) / CE_WARPS;
      if (p->edges_full && full_bytes <= (size_t)optin_ce - 2048) {
        // the whole JM in shared memory: no barrier inside the control loop
        static bool fattr = false;
        if (!fattr) {
          KFBI_CUDA(cudaFuncSetAttribute(corr_edges_full_kernel<T, E>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, optin_ce - 2048),
                    "jumps-and-corrections");
          fattr = true;
        }
        return launch(p, KFBI_K_JUMPS, s, [&] {
          corr_edges_full_kernel<T, E><<<blocks, CE_WARPS * 32, full_bytes, s>>>(
              ea, static_cast<const T *>(jm), static_cast<T *>(jv), done);
        });
      }
      return launch(p, KFBI_K_JUMPS, s, [&] {
        corr_edges_smem_kernel<T, E><<<blocks, CE_WARPS * 32, 0, s>>>(
            ea, static_cast<const T *>(jm), static_cast<T *>(jv), done);
      });
    };
    if (pw <= 2) return go(std::integral_constant<int, 2>());
    return go(std::integral_constant<int, 4>());
  }
  const int wave_warps = sms * 2 * 8;
  int per_warp = (p->n_edges + wave_warps - 1) / wave_warps;
  if (per_warp > EW) per_warp = EW;
  if (per_warp < 1) per_warp = 1;
  EdgeArgs ea{p->n_edges, p->n_ctl, p->w_ld, per_warp, p->W.p, p->edge_axis.p};
  const int warps = (p->n_edges + per_warp - 1) / per_warp;
  const int blocks = (warps + 7) / 8;
  if (p->n_edges == 0) return KFBI_OK;
  return launch(p, KFBI_K_JUMPS, s, [&] {
    corr_edges_kernel<T, EW, U><<<blocks, 256, 0, s>>>(ea, static_cast<const T *>(jm),
                                                       static_cast<T *>(jv), done);
  });
}

kfbi_status read_norm(kfbi_plan *p, cudaStream_t s, double *out) {
  KFBI_CUDA(cudaMemcpyAsync(p->red_host, p->red.p, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s), "rhs-update");
  KFBI_CUDA(cudaStreamSynchronize(s), "rhs-update");
  long long bits = (long long)p->red_host[0];
  double v;
  std::memcpy(&v, &bits, sizeof v);
  if (out) *out = v;
  return KFBI_OK;
}

int elem_blocks(long n) {
  long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

// grid of the two-elements-per-step passes (elementwise_pairs)
int pair_blocks(long n) {
  long b = (n + 1023) / 1024;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

bool aligned16(std::initializer_list<const void *> ptrs) {
  for (const void *q : ptrs)
    if (q && (reinterpret_cast<uintptr_t>(q) & 15)) return false;
  return true;
}

// One Richardson sweep, every kernel guarded by the device `done` flag.
template <typename T>
kfbi_status sweep(kfbi_plan *p, const kfbi_bvp *b, cudaStream_t s) {
  const int *done = &p->st.p->done;
  const bool dir = b->bc_kind == 0;
  // Dirichlet: density = phi = [u]; Neumann: density = psi = [u_n] (bvp.py:313-317)
  KFBI_TRY(jumps_T<T>(p, b->kappa_re, b->kappa_im, dir ? b->density : nullptr,
                      dir ? nullptr : b->density, b->f_gamma, b->f_gamma_sign, p->jm.p, done, s));
  KFBI_TRY(edges_T<T>(p, p->jm.p, p->jv.p, done, s));
  KFBI_TRY(box_dispatch(p, std::is_same<T, double2>::value ? KFBI_C128 : KFBI_F64, b->kappa_re,
                        b->kappa_im, b->F, b->F_sign, p->jv.p, b->u, done, s, b->box_bc));
  ExtractArgs x = extract_args(p, !dir);
  const int blocks = (p->n_ctl + 255) / 256;
  return launch(p, KFBI_K_DENSITY, s, [&] {
    extract_update_kernel<T><<<blocks, 256, 0, s>>>(
        x, static_cast<const T *>(b->u), reinterpret_cast<const T *>(p->jm.p),
        static_cast<const T *>(b->g), static_cast<T *>(b->density), static_cast<T *>(b->trace_u),
        static_cast<T *>(b->trace_un), b->gamma, dir ? 1 : 0, p->st.p, p->history.p);
  });
}


kfbi_status ensure_op_scratch(kfbi_plan *p) {
  const size_t n = (size_t)p->n_ctl;
  cudaError_t e = cudaSuccess;
  DevBuf<double2> *bufs[] = {&p->phi0, &p->phi_prev, &p->trace1, &p->trace_tmp, &p->zvec, &p->evec};
  for (auto *b : bufs)
    if (e == cudaSuccess) e = b->ensure(n);
  if (e == cudaSuccess) e = p->out3.ensure(3 * n);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("operator scratch: ") + cudaGetErrorString(e));
  return KFBI_OK;
}

kfbi_status ensure_async_scratch(kfbi_plan *p) {
  cudaError_t e = p->phik1.ensure((size_t)p->n_ctl);
  if (e == cudaSuccess) e = p->skip.ensure(1);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("async scratch: ") + cudaGetErrorString(e));
  return KFBI_OK;
}

// Column p of T = trace of the pipeline applied to e_p with F = 0, f_gamma = 0.
bool facr_trace_applies(kfbi_plan *p, double kre, double kim, bool cplx, int bc_kind, int box_bc);

template <typename T>
kfbi_status build_operator_T(kfbi_plan *p, double kre, double kim, int bc_kind, int box_bc,
                             cudaStream_t s) {
  constexpr bool CPLX = std::is_same<T, double2>::value;
  const int n = p->n_ctl;
  const size_t nf = (size_t)(p->m + 1) * (p->m + 1);
  KFBI_TRY(ensure_op_scratch(p));
  cudaError_t e = p->Top.ensure((size_t)n * n);
  if (e == cudaSuccess) e = p->ufield.ensure(nf);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("operator allocation: ") + cudaGetErrorString(e));
  p->op_valid = false;
  T *z = reinterpret_cast<T *>(p->zvec.p), *ev = reinterpret_cast<T *>(p->evec.p);
  T *out = reinterpret_cast<T *>(p->out3.p), *Top = reinterpret_cast<T *>(p->Top.p);
  KFBI_CUDA(cudaMemsetAsync(z, 0, n * sizeof(T), s), "jumps-and-corrections");
  const bool dir = bc_kind == 0;
  ExtractArgs x = extract_args(p, !dir);
  const int eb = (n + 255) / 256;
  const bool timing = p->timing;
  p->timing = false;
  const bool sparse = facr_trace_applies(p, kre, kim, CPLX, bc_kind, box_bc);
  kfbi_status st = KFBI_OK;
  for (int col = 0; col < n && st == KFBI_OK; ++col) {
    st = launch(p, KFBI_K_JUMPS, s, [&] { unit_vector_kernel<T><<<eb, 256, 0, s>>>(ev, n, col); });
    if (st == KFBI_OK)
      st = jumps_T<T>(p, kre, kim, dir ? ev : nullptr, dir ? nullptr : ev, z, 1.0, p->jm.p, nullptr, s);
    if (st == KFBI_OK) st = edges_T<T>(p, p->jm.p, p->jv.p, nullptr, s);
    if (st == KFBI_OK) {
      if (sparse) {                              // only the trace is needed: stencil chunks of the odd rows
        BoxArgs a = box_args(p, kre, kim, nullptr);
        a.npl = CPLX ? p->m / 2 : p->m / 4;
        a.oc_list = p->oc_list.p;
        a.n_oc = p->n_oc;
        a.row_need = p->need_trace.p;
        CorrArgs<T> c = corr_args<T>(p, reinterpret_cast<const T *>(p->jv.p));
        st = box_passes_reg<CPLX>(p, a, nullptr, 1.0, c, p->ufield.p, s);
      } else {
        st = box_dispatch(p, CPLX ? KFBI_C128 : KFBI_F64, kre, kim, nullptr, 1.0, p->jv.p, p->ufield.p,
                          nullptr, s, box_bc);
      }
    }
    if (st == KFBI_OK)
      st = launch(p, KFBI_K_EXTRACT, s, [&] {
        extract_kernel<T><<<eb, 256, 0, s>>>(x, reinterpret_cast<const T *>(p->ufield.p),
                                             reinterpret_cast<const T *>(p->jm.p), out);
      });
    if (st == KFBI_OK)
      st = launch(p, KFBI_K_EXTRACT, s, [&] {
        op_column_kernel<T><<<eb, 256, 0, s>>>(n, col, out, p->normal.p, dir ? 0 : 1, Top);
      });
  }
  p->timing = timing;
  KFBI_TRY(st);
  KFBI_CUDA(cudaStreamSynchronize(s), "extract-traces");
  p->op_valid = true;
  p->op_dtype = CPLX ? KFBI_C128 : KFBI_F64;
  p->op_kre = kre;
  p->op_kim = kim;
  p->op_bc = bc_kind * 2 + box_bc;
  return KFBI_OK;
}

// The on-chip operator sweeps give each CTA (one per SM) R = ceil(n / SMs)
// rows of T, rounded up to even; the sweep kernels cover R <= 32 rows (one
// row per lane, or row pairs on half-warps).  Larger n_ctl must use the
// pipeline form.
int op_sms(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms > 0 ? sms : 1;
}
int op_max_ctl(kfbi_plan *p) { return 32 * op_sms(p->device); }

// All operator sweeps of one solve: one cooperative launch (op_solve_kernel),
// T resident on chip (registers + shared memory) across the sweeps.
template <typename T>
kfbi_status op_solve(kfbi_plan *p, const kfbi_bvp *b, cudaStream_t s) {
  constexpr int K = OpTune<T>::K;
  static int smem_optin = 0, sms = 0;
  if (!smem_optin) {
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    KFBI_CUDA(cudaFuncSetAttribute(op_solve_kernel<T, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem_optin - 1024), "density-update");
  }
  const int n = p->n_ctl;
  int rows = (n + sms - 1) / sms;
  rows += rows & 1;                       // even: 16-byte row pairs (pair kernel)
  if (rows > 32)
    return fail(KFBI_E_CONFIG, "operator form: n_ctl = " + std::to_string(n) + " exceeds 32 rows per SM (" +
                                   std::to_string(32 * sms) + " controls); use the pipeline form");
  const int grid = (n + rows - 1) / rows;
  const size_t fixed = op_smem_fixed<T>(n);
  const size_t avail = (size_t)(smem_optin - 1024) > fixed ? (size_t)(smem_optin - 1024) - fixed : 0;
  const int creg = n < OP_WARPS * K ? n : OP_WARPS * K;
  size_t cs = avail / ((size_t)rows * sizeof(T));
  if (cs > (size_t)(n - creg)) cs = (size_t)(n - creg);
  const size_t smem = fixed + cs * rows * sizeof(T);
  if (fixed > (size_t)(smem_optin - 1024))
    return fail(KFBI_E_CONFIG, "operator form: n_ctl too large for the on-chip sweep kernel");
  unsigned long long *slots = p->red.p + 4;        // [3] maxima + the barrier counter
  KFBI_CUDA(cudaMemsetAsync(slots, 0, 4 * sizeof(unsigned long long), s), "density-update");
  OpSolveArgs a;
  a.n = n;
  a.first_idx = 1;
  a.max_iter = b->max_iter;
  a.gamma = b->gamma;
  a.tol = b->tol;
  a.st = p->st.p;
  a.history = p->history.p;
  a.slots = slots;
  a.bar = reinterpret_cast<unsigned int *>(slots + 3);
  a.rows = rows;
  a.smem_cols = (int)cs;
  const T *Tcm = reinterpret_cast<const T *>(p->Top.p);
  T *A = static_cast<T *>(b->density), *B = reinterpret_cast<T *>(p->phi_prev.p);
  const T *phi0 = reinterpret_cast<const T *>(p->phi0.p);
  const T *tr1 = reinterpret_cast<const T *>(p->trace1.p);
  const T *g = static_cast<const T *>(b->g);
  void *args[] = {&a, (void *)&Tcm, &A, &B, (void *)&phi0, (void *)&tr1, (void *)&g};
  // small n: all sweeps in one CTA, no grid barrier (op_solve_cta_kernel)
  if (n <= 160 && op_cta_smem<T>(n) <= (size_t)(smem_optin - 1024) && p->op_cta) {
    static bool cta_attr = false;
    if (!cta_attr) {
      KFBI_CUDA(cudaFuncSetAttribute(op_solve_cta_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem_optin - 1024), "density-update");
      cta_attr = true;
    }
    const size_t smc = op_cta_smem<T>(n);
    return launch(p, KFBI_K_DENSITY, s, [&] {
      op_solve_cta_kernel<T><<<1, OPC_THREADS, smc, s>>>(a, Tcm, A, B, phi0, tr1, g);
    });
  }
  if constexpr (std::is_same<T, double>::value) {
    // two rows per lane (16-byte pairs) when n and R are even
    constexpr int K2 = K / 2;
    if (n % 2 == 0 && rows % 2 == 0) {
      static bool pair_attr = false;
      if (!pair_attr) {
        KFBI_CUDA(cudaFuncSetAttribute(op_solve_pair_kernel<K2, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - 1024),
                  "density-update");
        KFBI_CUDA(cudaFuncSetAttribute(op_solve_pair_kernel<K2, 3>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - 1024),
                  "density-update");
        pair_attr = true;
      }
      // three column groups per warp when a CTA owns <= 20 rows (30 busy lanes
      // instead of rows / 2 of 32); the register-cached columns grow with G
      const int G = rows <= 20 ? 3 : 2;
      const int cregG = n < G * OP_WARPS * K2 ? n : G * OP_WARPS * K2;
      size_t csG = avail / ((size_t)rows * sizeof(T));
      if (csG > (size_t)(n - cregG)) csG = (size_t)(n - cregG);
      a.smem_cols = (int)csG;
      const size_t smemG = fixed + csG * rows * sizeof(T);
      const void *fn = G == 3 ? (const void *)op_solve_pair_kernel<K2, 3> : (const void *)op_solve_pair_kernel<K2, 2>;
      return launch(p, KFBI_K_DENSITY, s, [&] {
        return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(OP_THREADS), args, smemG, s);
      });
    }
  }
  if constexpr (std::is_same<T, double2>::value) {
    // complex rows on half-warps (16 busy lanes) when a CTA owns <= 16 rows
    if (rows <= 16) {
      constexpr int KH = KFBI_OP_K_HALF;
      static bool half_attr = false;
      if (!half_attr) {
        KFBI_CUDA(cudaFuncSetAttribute(op_solve_half_kernel<KH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_optin - 1024), "density-update");
        half_attr = true;
      }
      // twice the register-cached columns per row set: re-split the rest
      const int creg2 = n < 2 * OP_WARPS * KH ? n : 2 * OP_WARPS * KH;
      size_t cs2 = avail / ((size_t)rows * sizeof(T));
      if (cs2 > (size_t)(n - creg2)) cs2 = (size_t)(n - creg2);
      a.smem_cols = (int)cs2;
      const size_t smem2 = fixed + cs2 * rows * sizeof(T);
      return launch(p, KFBI_K_DENSITY, s, [&] {
        return cudaLaunchCooperativeKernel((const void *)op_solve_half_kernel<KH>, dim3(grid),
                                           dim3(OP_THREADS), args, smem2, s);
      });
    }
  }
  return launch(p, KFBI_K_DENSITY, s, [&] {
    cudaLaunchCooperativeKernel((const void *)op_solve_kernel<T, K>, dim3(grid), dim3(OP_THREADS), args,
                                smem, s);
  });
}

// A trace-only sweep through the FACR box solve (sweep 1 of the operator
// form, every sweep of the pipeline form) with only the stencil chunks of the
// odd rows (rows_odd_facr_sparse): the even rows come out whole, the odd rows
// only where the six-point stencils read them; the field of the converging
// sweep comes from one full pipeline (final_pipeline) from its start density.
bool facr_trace_applies(kfbi_plan *p, double kre, double kim, bool cplx, int bc_kind, int box_bc) {
  if (!p->facr_trace || !p->facr || p->n_oc <= 0 || bc_kind != 0 || box_bc != KFBI_DIRICHLET_ZERO)
    return false;
  if (!col_use_tri(p, kre, kim)) return false;
  return p->m >= 512 && (p->m <= 8192 || (!cplx && p->m == 16384));
}

bool facr_trace_ok(kfbi_plan *p, const kfbi_bvp *b) {
  return facr_trace_applies(p, b->kappa_re, b->kappa_im, b->dtype == KFBI_C128, b->bc_kind, b->box_bc);
}

template <typename T>
kfbi_status sweep1_facr_trace(kfbi_plan *p, const kfbi_bvp *b, cudaStream_t s) {
  constexpr bool CPLX = std::is_same<T, double2>::value;
  const int *done = &p->st.p->done;
  KFBI_TRY(jumps_T<T>(p, b->kappa_re, b->kappa_im, b->density, nullptr, b->f_gamma, b->f_gamma_sign,
                      p->jm.p, done, s));
  KFBI_TRY(edges_T<T>(p, p->jm.p, p->jv.p, done, s));
  BoxArgs a = box_args(p, b->kappa_re, b->kappa_im, done);
  a.npl = CPLX ? p->m / 2 : p->m / 4;
  a.oc_list = p->oc_list.p;
  a.n_oc = p->n_oc;
  a.row_need = p->need_trace.p;
  CorrArgs<T> c = corr_args<T>(p, reinterpret_cast<const T *>(p->jv.p));
  KFBI_TRY(box_passes_reg<CPLX>(p, a, b->F, b->F_sign, c, b->u, s));
  ExtractArgs x = extract_args(p, false);
  const int blocks = (p->n_ctl + 255) / 256;
  return launch(p, KFBI_K_DENSITY, s, [&] {
    extract_update_kernel<T><<<blocks, 256, 0, s>>>(
        x, static_cast<const T *>(b->u), reinterpret_cast<const T *>(p->jm.p),
        static_cast<const T *>(b->g), static_cast<T *>(b->density), static_cast<T *>(b->trace_u),
        static_cast<T *>(b->trace_un), b->gamma, 1, p->st.p, p->history.p);
  });
}

// Sweep 1 of the operator form when only its trace is needed (Dirichlet,
// one slab): rows_fwd + column stage, then the inverse row transform only at
// the stencil nodes (stencil_eval_kernel) instead of the whole field; the
// extraction and density update read those values (the slab update kernel).
bool trace_sweep_ok(kfbi_plan *p, const kfbi_bvp *b) {
  // one grid row per CTA, 16 elements per thread: 512 <= M <= 8192
  return p->trace_sweep && b->bc_kind == 0 && b->box_bc == KFBI_DIRICHLET_ZERO && p->sn_nrows > 0 &&
         p->m >= 512 && p->m <= 8192;
}

template <typename T>
kfbi_status sweep1_trace(kfbi_plan *p, const kfbi_bvp *b, cudaStream_t s) {
  constexpr bool CPLX = std::is_same<T, double2>::value;
  const int *done = &p->st.p->done;
  KFBI_TRY(jumps_T<T>(p, b->kappa_re, b->kappa_im, b->density, nullptr, b->f_gamma, b->f_gamma_sign,
                      p->jm.p, done, s));
  KFBI_TRY(edges_T<T>(p, p->jm.p, p->jv.p, done, s));
  BoxArgs a = box_args(p, b->kappa_re, b->kappa_im, done);
  a.npl = CPLX ? p->m / 2 : p->m / 4;
  CorrArgs<T> c = corr_args<T>(p, reinterpret_cast<const T *>(p->jv.p));
  KFBI_TRY(box_passes_reg<CPLX>(p, a, b->F, b->F_sign, c, nullptr, s, 3));
  T *nv = reinterpret_cast<T *>(p->sn_vals.p);
  KFBI_TRY(launch(p, KFBI_K_EXTRACT, s, [&] {
    stencil_eval_kernel<CPLX><<<p->sn_nrows, p->m / SEVAL_E, 0, s>>>(a, p->sn_rows.p, p->sn_rowptr.p,
                                                                     p->sn_cols.p, nv);
  }));
  T *v13 = reinterpret_cast<T *>(p->sn_v13.p);
  const int blocks = (p->n_ctl + 255) / 256;
  KFBI_TRY(launch(p, KFBI_K_EXTRACT, s, [&] {
    stencil_vals_kernel<T><<<blocks, 256, 0, s>>>(p->n_ctl, p->sn_map.p, nv, v13);
  }));
  ExtractArgs x = extract_args(p, false);
  return launch(p, KFBI_K_DENSITY, s, [&] {
    extract_update_vals_kernel<T><<<blocks, 256, 0, s>>>(
        x, v13, reinterpret_cast<const T *>(p->jm.p), static_cast<const T *>(b->g),
        static_cast<T *>(b->density), static_cast<T *>(b->trace_u), static_cast<T *>(b->trace_un),
        b->gamma, 1, p->st.p, p->history.p);
  });
}

// Full pipeline from the density before the converging update: the field and
// traces the reference returns (bvp.py:319-323, 336-344).
template <typename T>
kfbi_status final_pipeline(kfbi_plan *p, const kfbi_bvp *b, const void *phi_before, cudaStream_t s,
                           const int *skip = nullptr) {
  constexpr bool CPLX = std::is_same<T, double2>::value;
  const int n = p->n_ctl;
  const bool dir = b->bc_kind == 0;
  KFBI_TRY(jumps_T<T>(p, b->kappa_re, b->kappa_im, dir ? phi_before : nullptr,
                      dir ? nullptr : phi_before, b->f_gamma, b->f_gamma_sign, p->jm.p, skip, s));
  KFBI_TRY(edges_T<T>(p, p->jm.p, p->jv.p, skip, s));
  if (b->field_chunks && p->n_fc > 0 &&
      facr_trace_applies(p, b->kappa_re, b->kappa_im, CPLX, b->bc_kind, b->box_bc)) {
    // the caller reads the field only at the interior and stencil nodes
    // (kfbi_plan_set_field_chunks): odd rows only at their chunks
    BoxArgs a = box_args(p, b->kappa_re, b->kappa_im, skip);
    a.npl = CPLX ? p->m / 2 : p->m / 4;
    a.span = p->fc_span.p;
    a.row_need = p->need_field.p;
    CorrArgs<T> c = corr_args<T>(p, reinterpret_cast<const T *>(p->jv.p));
    KFBI_TRY(box_passes_reg<CPLX>(p, a, b->F, b->F_sign, c, b->u, s));
  } else {
    KFBI_TRY(box_dispatch(p, CPLX ? KFBI_C128 : KFBI_F64, b->kappa_re, b->kappa_im, b->F, b->F_sign,
                          p->jv.p, b->u, skip, s, b->box_bc));
  }
  ExtractArgs x = extract_args(p, !dir);
  return launch(p, KFBI_K_EXTRACT, s, [&] {
    extract_traces_kernel<T><<<(n + 255) / 256, 256, 0, s>>>(
        x, static_cast<const T *>(b->u), reinterpret_cast<const T *>(p->jm.p),
        static_cast<T *>(b->trace_u), static_cast<T *>(b->trace_un), skip);
  });
}

// w = T v: the pipeline with F = 0, f_gamma = 0 applied to the density v
// (the column map of build_operator_T), or the plan's explicit operator.
template <typename T>
kfbi_status gm_matvec(kfbi_plan *p, const kfbi_bvp *b, const T *v, T *w, bool op, cudaStream_t s) {
  constexpr bool CPLX = std::is_same<T, double2>::value;
  const int n = p->n_ctl;
  GmresState *st = p->gm_st.p;
  const int *done = &st->done;
  if (op) {
    T *part = reinterpret_cast<T *>(p->gm_tr.p);
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
      gm_gemv_kernel<T><<<dim3((n + GM_T - 1) / GM_T, GM_JS), GM_T, 0, s>>>(
          n, reinterpret_cast<const T *>(p->Top.p), v, part, st);
    }));
    return launch(p, KFBI_K_DENSITY, s, [&] {
      gm_gemv_sum_kernel<T><<<(n + GM_T - 1) / GM_T, GM_T, 0, s>>>(n, part, w, st);
    });
  }
  const bool dir = b->bc_kind == 0;
  T *z = reinterpret_cast<T *>(p->zvec.p);
  KFBI_TRY(jumps_T<T>(p, b->kappa_re, b->kappa_im, dir ? v : nullptr, dir ? nullptr : v, z, 1.0, p->jm.p,
                      done, s));
  KFBI_TRY(edges_T<T>(p, p->jm.p, p->jv.p, done, s));
  KFBI_TRY(box_dispatch(p, CPLX ? KFBI_C128 : KFBI_F64, b->kappa_re, b->kappa_im, nullptr, 1.0, p->jv.p,
                        p->ufield.p, done, s, b->box_bc));
  ExtractArgs x = extract_args(p, !dir);
  T *other = reinterpret_cast<T *>(p->gm_tr.p);
  return launch(p, KFBI_K_EXTRACT, s, [&] {
    extract_traces_kernel<T><<<(n + 255) / 256, 256, 0, s>>>(
        x, reinterpret_cast<const T *>(p->ufield.p), reinterpret_cast<const T *>(p->jm.p),
        dir ? w : other, dir ? other : w, done);
  });
}

// Restarted GMRES(m) on T phi = g - t_F (gmres.cuh); one host sync per cycle.
template <typename T>
kfbi_status gmres_T(kfbi_plan *p, const kfbi_bvp *b, int m, kfbi_bvp_result *res, cudaStream_t s) {
  const int n = p->n_ctl;
  const size_t nf = (size_t)(p->m + 1) * (p->m + 1);
  const bool op = b->use_operator != 0;
  cudaError_t e = cudaSuccess;
  DevBuf<double2> *vb[] = {&p->gm_w, &p->gm_g, &p->gm_sn, &p->gm_y};
  for (auto *q : vb)
    if (e == cudaSuccess) e = q->ensure((size_t)m + 1 > (size_t)n ? (size_t)m + 1 : (size_t)n);
  if (e == cudaSuccess) e = p->gm_V.ensure((size_t)(m + 1) * n);
  if (e == cudaSuccess) e = p->gm_H.ensure((size_t)(m + 1) * m);
  if (e == cudaSuccess) e = p->gm_part.ensure((size_t)(m + 1) * GM_NB);
  if (e == cudaSuccess) e = p->gm_tr.ensure((size_t)GM_JS * n > (size_t)n ? (size_t)GM_JS * n : (size_t)n);
  if (e == cudaSuccess) e = p->gm_cs.ensure((size_t)m + 1);
  if (e == cudaSuccess) e = p->gm_np.ensure(GM_NB);
  if (e == cudaSuccess) e = p->gm_st.ensure(1);
  if (e == cudaSuccess) e = p->ufield.ensure(nf);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("gmres scratch: ") + cudaGetErrorString(e));
  KFBI_TRY(ensure_op_scratch(p));
  KFBI_CUDA(cudaMemsetAsync(p->zvec.p, 0, n * sizeof(double2), s), "density-update");
  T *V = reinterpret_cast<T *>(p->gm_V.p), *w = reinterpret_cast<T *>(p->gm_w.p);
  T *H = reinterpret_cast<T *>(p->gm_H.p), *sn = reinterpret_cast<T *>(p->gm_sn.p);
  T *gv = reinterpret_cast<T *>(p->gm_g.p), *y = reinterpret_cast<T *>(p->gm_y.p);
  T *part = reinterpret_cast<T *>(p->gm_part.p), *x = static_cast<T *>(b->density);
  GmresState *st = p->gm_st.p;
  double *np = p->gm_np.p, *cs = p->gm_cs.p;
  const bool dir = b->bc_kind == 0;
  KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_init_kernel<<<1, 1, 0, s>>>(st, b->max_iter, b->tol, b->gamma); }));
  GmresState hs{};
  int cycles = 0;
  for (;;) {
    // r0 = g - trace(x): one full sweep (F, f_gamma) from the current density
    KFBI_TRY(final_pipeline<T>(p, b, x, s));
    const T *tr = static_cast<const T *>(dir ? b->trace_u : b->trace_un);
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
      gm_start_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, static_cast<const T *>(b->g), tr, w, np, st);
    }));
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_begin_kernel<T><<<1, 32, 0, s>>>(np, gv, st, p->history.p); }));
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_scale_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, w, V, st); }));
    for (int j = 0; j < m; ++j) {
      KFBI_TRY(gm_matvec<T>(p, b, V + (size_t)j * n, w, op, s));
      for (int pass = 0; pass < 2; ++pass) {       // classical Gram-Schmidt, twice
        KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_dots_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, j, V, w, part, st); }));
        KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
          gm_orth_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, j, m, V, w, part, H, pass, np, st);
        }));
      }
      KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
        gm_givens_kernel<T><<<1, 32, 0, s>>>(j, m, np, H, cs, sn, gv, st, p->history.p);
      }));
      KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
        gm_scale_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, w, V + (size_t)(j + 1) * n, st);
      }));
    }
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_backsolve_kernel<T><<<1, 32, 0, s>>>(m, H, gv, y, st); }));
    KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { gm_update_kernel<T><<<GM_NB, GM_T, 0, s>>>(n, V, y, x, st); }));
    KFBI_CUDA(cudaMemcpyAsync(&hs, st, sizeof(GmresState), cudaMemcpyDeviceToHost, s), "density-update");
    KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
    ++cycles;
    if (hs.done || hs.iters >= b->max_iter) break;
    // next cycle: rotation state restarts, the density carries over
  }
  // the returned field and traces: one full sweep from the final density
  KFBI_TRY(final_pipeline<T>(p, b, x, s));
  res->iterations = hs.iters + cycles + 1;        // matvecs + full sweeps
  res->converged = hs.done == 1 ? 1 : 0;
  res->residual = b->gamma * hs.resid;
  if (res->history) {
    const int nh = hs.iters < b->max_iter ? hs.iters : b->max_iter;
    if (nh > 0)
      KFBI_CUDA(cudaMemcpy(res->history, p->history.p, nh * sizeof(double), cudaMemcpyDeviceToHost),
                "density-update");
  }
  KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
  if (hs.done != 1)
    return fail(KFBI_E_NOCONV, "GMRES did not reach tol within max_iter matvecs (last gamma*||r|| " +
                                   std::to_string(b->gamma * hs.resid) + ")");
  return KFBI_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

const char *kfbi_last_error(void) { return g_last_error.c_str(); }
const char *kfbi_version(void) { return "kfbi_b200 0.1.0 (sm_100a)"; }

kfbi_status kfbi_plan_create(const kfbi_grid_desc *desc, kfbi_plan **out) {
  if (!desc || !out) return fail(KFBI_E_CONFIG, "null argument");
  const int m = desc->m;
  if (m < 16 || (m & (m - 1)) != 0) return fail(KFBI_E_GRID, "M must be a power of two and >= 16");
  if (m > 16384) return fail(KFBI_E_CONFIG, "this build supports M <= 16384");
  if (!(desc->h > 0)) return fail(KFBI_E_GRID, "grid spacing must be positive");
  kfbi_plan *p = new kfbi_plan();
  p->device = desc->device;
  p->m = m;
  p->logm = ilog2(m);
  p->h = desc->h;
  {
    const char *f = std::getenv("KFBI_FACR");      // "0": three-pass box solves by default
    if (f && f[0] == '0') p->facr = false;
    const char *es = std::getenv("KFBI_EDGES_SMEM");
    if (es && es[0] == '0') p->edges_smem = false;
    const char *oc = std::getenv("KFBI_OP_CTA");
    if (oc && oc[0] == '0') p->op_cta = false;
    const char *ef = std::getenv("KFBI_EDGES_FULL");
    if (ef && ef[0] == '0') p->edges_full = false;
    const char *ft = std::getenv("KFBI_FACR_TRACE");
    if (ft && ft[0] == '0') p->facr_trace = false;
  }
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) {
    delete p;
    return fail(KFBI_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  // lambda_p exactly as boxsolve.py:43 evaluates it in double:
  // (2 cos(p pi / m) - 2) / h^2
  std::vector<double> lam(m + 1, 0.0);
  for (int q = 1; q <= m; ++q) {      // p = m only for the neumann-zero closure
    double ang = (double)q * M_PI / (double)m;
    lam[q] = (2.0 * std::cos(ang) - 2.0) / (desc->h * desc->h);
  }
  // register engine tables: exp(-2 pi i q / m) and sin(pi j / m), q, j < m
  std::vector<double2> twg(m);
  std::vector<double> sinv(m);
  for (int q = 0; q < m; ++q) {
    long double ang = 3.14159265358979323846264338327950288L * (long double)q / (long double)m;
    twg[q] = make_double2((double)cosl(2.0L * ang), (double)-sinl(2.0L * ang));
    sinv[q] = (double)sinl(ang);
  }
  if ((e = upload(p->twg, twg.data(), twg.size())) != cudaSuccess ||
      (e = upload(p->sinv, sinv.data(), sinv.size())) != cudaSuccess ||
      (e = upload(p->lam, lam.data(), lam.size())) != cudaSuccess ||
      (e = p->panels.ensure((size_t)(m + 2) * (m + 2))) != cudaSuccess ||
      (e = p->rowz.ensure((size_t)m / 2 + 2)) != cudaSuccess ||
      (e = p->st.ensure(1)) != cudaSuccess || (e = p->red.ensure(8)) != cudaSuccess) {
    kfbi_plan_destroy(p);
    return fail(KFBI_E_CUDA, std::string("plan allocation: ") + cudaGetErrorString(e));
  }
  cudaMemset(p->panels.p, 0, (size_t)(m + 2) * (m + 2) * sizeof(double2));
  cudaMallocHost(&p->st_host, sizeof(RichState));
  cudaMallocHost(&p->red_host, 4 * sizeof(unsigned long long));
  *out = p;
  return KFBI_OK;
}

kfbi_status kfbi_slab_panel_bytes(kfbi_plan *p, int32_t dtype, int32_t nranks, int64_t *bytes) {
  KFBI_TRY(check_plan(p));
  if (!bytes || nranks < 1) return fail(KFBI_E_CONFIG, "slab: bad argument");
  *bytes = (int64_t)(p->m / nranks) * p->m * (dtype == KFBI_C128 ? 16 : 8);
  return KFBI_OK;
}

kfbi_status kfbi_slab_tri_bytes(kfbi_plan *p, int32_t dtype, int32_t nranks, int64_t *agg_bytes,
                                int64_t *flag_bytes) {
  KFBI_TRY(check_plan(p));
  if (!agg_bytes || !flag_bytes || nranks < 1 || nranks > KFBI_MAX_PEERS)
    return fail(KFBI_E_CONFIG, "slab: bad argument");
  // units x P x NH x 3 double2 (NH x units = 2 x panels either way), units x P flags
  const int64_t npl = dtype == KFBI_C128 ? p->m / 2 : p->m / 4;
  *agg_bytes = 2 * npl * nranks * 3 * 16;
  *flag_bytes = 2 * npl * nranks * 8;
  return KFBI_OK;
}

kfbi_status kfbi_slab_cols_tri(kfbi_plan *p, int32_t dtype, int32_t nranks, int32_t rank, double kre,
                               double kim, void *panels, const kfbi_tri_dist *d, void *stream) {
  KFBI_TRY(check_plan(p));
  if (!d || (!panels && !d->virt)) return fail(KFBI_E_CONFIG, "slab: null argument");
  const bool cplx = dtype == KFBI_C128;
  if (!cplx && kim != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  if (nranks != d->nranks || rank != d->rank || nranks < 1 || nranks > KFBI_MAX_PEERS ||
      (nranks & (nranks - 1)) != 0 || rank < 0 || rank >= nranks || p->m / nranks < 16)
    return fail(KFBI_E_CONFIG, "slab column stage: nranks a power of two <= 8, M / nranks >= 16");
  for (int h = 0; h < nranks; ++h)
    if (!d->agg[h] || !d->flags[h] || (d->virt && !d->panels[h]))
      return fail(KFBI_E_CONFIG, "slab column stage: null peer buffer");
  if (d->epoch < 1) return fail(KFBI_E_CONFIG, "slab column stage: epoch must be >= 1");
  BoxArgs a = box_args(p, kre, kim, nullptr);
  a.rows = p->m / nranks;
  a.row0 = rank * a.rows;
  a.panels = panels;
  const int logr = ilog2(a.rows);
  return box_cols_dist(p, cplx, logr, a, d, (cudaStream_t)stream);
}

kfbi_status kfbi_slab_rows_fwd(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, const void *rhs,
                               double sign, const void *jv, void *panels, void *stream) {
  return slab_pass(p, dtype, sl, 1, 0.0, 0.0, rhs, sign, jv, panels, nullptr, stream);
}

kfbi_status kfbi_slab_cols(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, double kappa_re,
                           double kappa_im, void *panels, void *stream) {
  return slab_pass(p, dtype, sl, 2, kappa_re, kappa_im, nullptr, 1.0, nullptr, panels, nullptr, stream);
}

kfbi_status kfbi_slab_rows_inv(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, const void *panels,
                               void *u, void *stream) {
  return slab_pass(p, dtype, sl, 4, 0.0, 0.0, nullptr, 1.0, nullptr, const_cast<void *>(panels), u,
                   stream);
}

kfbi_status kfbi_slab_rows_fwd_p2p(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, const void *rhs,
                                   double sign, const void *jv, void *const *peer_panels,
                                   void *stream) {
  if (!peer_panels) return fail(KFBI_E_CONFIG, "slab p2p: null peer table");
  return slab_pass(p, dtype, sl, 1, 0.0, 0.0, rhs, sign, jv, nullptr, nullptr, stream, peer_panels);
}

kfbi_status kfbi_slab_cols_p2p(kfbi_plan *p, int32_t dtype, const kfbi_slab *sl, double kappa_re,
                               double kappa_im, const void *panels, void *const *peer_panels,
                               void *stream) {
  if (!peer_panels) return fail(KFBI_E_CONFIG, "slab p2p: null peer table");
  return slab_pass(p, dtype, sl, 2, kappa_re, kappa_im, nullptr, 1.0, nullptr,
                   const_cast<void *>(panels), nullptr, stream, peer_panels);
}

// ---- peer memory (CUDA IPC) and the peer-flag barrier ----

kfbi_status kfbi_ipc_alloc(int64_t bytes, void **ptr, void *handle) {
  if (!ptr || !handle || bytes <= 0) return fail(KFBI_E_CONFIG, "ipc: bad argument");
  KFBI_CUDA(cudaMalloc(ptr, (size_t)bytes), "ipc-alloc");
  KFBI_CUDA(cudaMemset(*ptr, 0, (size_t)bytes), "ipc-alloc");   // flags start at epoch 0
  KFBI_CUDA(cudaMemset(*ptr, 0, (size_t)bytes), "ipc-alloc");
  cudaIpcMemHandle_t h;
  KFBI_CUDA(cudaIpcGetMemHandle(&h, *ptr), "ipc-alloc");
  static_assert(sizeof(h) == KFBI_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  return KFBI_OK;
}

kfbi_status kfbi_ipc_free(void *ptr) {
  if (ptr) KFBI_CUDA(cudaFree(ptr), "ipc-free");
  return KFBI_OK;
}

kfbi_status kfbi_ipc_open(const void *handle, void **ptr) {
  if (!ptr || !handle) return fail(KFBI_E_CONFIG, "ipc: bad argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  KFBI_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc-open");
  return KFBI_OK;
}

kfbi_status kfbi_ipc_close(void *ptr) {
  if (ptr) KFBI_CUDA(cudaIpcCloseMemHandle(ptr), "ipc-close");
  return KFBI_OK;
}

kfbi_status kfbi_p2p_barrier(void *const *peer_flags, int32_t nranks, int32_t rank, int64_t epoch,
                             int64_t max_spins, int32_t *timed_out, void *stream) {
  if (!peer_flags || nranks < 1 || nranks > KFBI_MAX_PEERS || rank < 0 || rank >= nranks || epoch < 1)
    return fail(KFBI_E_CONFIG, "p2p barrier: bad argument");
  P2pFlags f;
  for (int h = 0; h < KFBI_MAX_PEERS; ++h) f.flags[h] = h < nranks ? (unsigned long long *)peer_flags[h] : nullptr;
  for (int h = 0; h < nranks; ++h)
    if (!f.flags[h]) return fail(KFBI_E_CONFIG, "p2p barrier: null flag buffer");
  p2p_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(f, nranks, rank,
                                                          (unsigned long long)epoch,
                                                          max_spins > 0 ? (long long)max_spins : (1ll << 28),
                                                          timed_out);
  KFBI_CUDA(cudaGetLastError(), "p2p-barrier");
  return KFBI_OK;
}

// ---- slab-decomposed Richardson sweep (dist.py SlabRichardson) ----
kfbi_status kfbi_edge_values(kfbi_plan *p, int32_t dtype, const void *jm, void *jv, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KFBI_C128) return edges_T<double2>(p, jm, jv, nullptr, s);
  return edges_T<double>(p, jm, jv, nullptr, s);
}

kfbi_status kfbi_slab_stencil_values(kfbi_plan *p, int32_t dtype, int32_t bc_kind, const kfbi_slab *sl,
                                     const void *u_slab, void *vals, void *stream) {
  KFBI_TRY(check_geo(p));
  if (!sl) return fail(KFBI_E_CONFIG, "slab: null argument");
  if (bc_kind == 1 && !p->has_os) return fail(KFBI_E_CONFIG, "one-sided extraction tables missing");
  BoxArgs a = box_args(p, 0.0, 0.0, nullptr);
  KFBI_TRY(slab_args(p, dtype == KFBI_C128, sl->nranks, sl->rank, a));
  ExtractArgs x = extract_args(p, bc_kind == 1);
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (p->n_ctl + 255) / 256;
  return launch(p, KFBI_K_EXTRACT, s, [&] {
    if (dtype == KFBI_C128)
      slab_stencil_kernel<double2><<<blocks, 256, 0, s>>>(x, a.row0, a.rows,
                                                          static_cast<const double2 *>(u_slab),
                                                          static_cast<double2 *>(vals));
    else
      slab_stencil_kernel<double><<<blocks, 256, 0, s>>>(x, a.row0, a.rows,
                                                         static_cast<const double *>(u_slab),
                                                         static_cast<double *>(vals));
  });
}

kfbi_status kfbi_rich_begin(kfbi_plan *p, int32_t max_iter, double tol, void *stream) {
  KFBI_TRY(check_geo(p));
  if (max_iter < 1) return fail(KFBI_E_CONFIG, "max iterations must be >= 1");
  cudaError_t e = p->history.ensure(max_iter);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, "history allocation failed");
  cudaStream_t s = (cudaStream_t)stream;
  return launch(p, KFBI_K_DENSITY, s, [&] { rich_init_kernel<<<1, 1, 0, s>>>(p->st.p, max_iter, tol); });
}

kfbi_status kfbi_slab_update(kfbi_plan *p, int32_t dtype, int32_t bc_kind, const void *vals,
                             const void *jm, const void *g, void *density, void *trace_u,
                             void *trace_un, double gamma, void *stream) {
  KFBI_TRY(check_geo(p));
  ExtractArgs x = extract_args(p, bc_kind == 1);
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (p->n_ctl + 255) / 256;
  return launch(p, KFBI_K_DENSITY, s, [&] {
    if (dtype == KFBI_C128)
      extract_update_vals_kernel<double2><<<blocks, 256, 0, s>>>(
          x, static_cast<const double2 *>(vals), static_cast<const double2 *>(jm),
          static_cast<const double2 *>(g), static_cast<double2 *>(density),
          static_cast<double2 *>(trace_u), static_cast<double2 *>(trace_un), gamma, bc_kind == 0,
          p->st.p, p->history.p);
    else
      extract_update_vals_kernel<double><<<blocks, 256, 0, s>>>(
          x, static_cast<const double *>(vals), static_cast<const double *>(jm),
          static_cast<const double *>(g), static_cast<double *>(density),
          static_cast<double *>(trace_u), static_cast<double *>(trace_un), gamma, bc_kind == 0,
          p->st.p, p->history.p);
  });
}

kfbi_status kfbi_rich_state(kfbi_plan *p, int32_t *iterations, int32_t *done, double *residual,
                            double *history, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemcpyAsync(p->st_host, p->st.p, sizeof(RichState), cudaMemcpyDeviceToHost, s),
            "density-update");
  KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
  if (iterations) *iterations = p->st_host->iters;
  if (done) *done = p->st_host->done;
  if (residual) *residual = p->st_host->last_res;
  if (history && p->st_host->iters > 0)
    KFBI_CUDA(cudaMemcpy(history, p->history.p, sizeof(double) * p->st_host->iters, cudaMemcpyDeviceToHost),
              "density-update");
  return KFBI_OK;
}

kfbi_status kfbi_plan_destroy(kfbi_plan *p) {
  if (!p) return KFBI_OK;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (auto &pe : p->pending) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  for (auto e : p->pool) cudaEventDestroy(e);
  p->lam.release(); p->panels.release(); p->twg.release(); p->sinv.release();
  p->W.release(); p->edge_theta_d.release(); p->ctl_theta_d.release(); p->spec.release();
  p->spec_part.release(); p->edge_perm.release(); p->spec_ctr.release(); p->edge_axis.release(); p->rec_edge.release(); p->group_start.release();
  p->group_node.release(); p->row_group.release(); p->stencil.release(); p->rec_d.release();
  p->rec_sigma.release(); p->deriv_col.release(); p->speed.release(); p->tangent.release();
  p->normal.release(); p->dtan_ds.release(); p->inv3.release(); p->ainv_rows.release();
  p->jcoef.release(); p->os_stencil.release(); p->os_rows.release(); p->os_fb.release(); p->d1.release(); p->psi_s.release(); p->jm.release(); p->jv.release();
  p->history.release(); p->st.release(); p->red.release();
  p->Top.release(); p->phi0.release(); p->phi_prev.release(); p->trace1.release();
  p->trace_tmp.release(); p->zvec.release(); p->evec.release(); p->out3.release();
  p->ufield.release(); p->phik1.release(); p->skip.release(); p->log.release();
  if (p->st_host) cudaFreeHost(p->st_host);
  if (p->red_host) cudaFreeHost(p->red_host);
  delete p;
  return KFBI_OK;
}

kfbi_status kfbi_box_solve(kfbi_plan *p, int32_t dtype, double kre, double kim, const void *rhs,
                           void *u, void *stream) {
  KFBI_TRY(check_plan(p));
  if (!rhs || !u) return fail(KFBI_E_CONFIG, "null field pointer");
  return box_dispatch(p, dtype, kre, kim, rhs, 1.0, nullptr, u, nullptr, (cudaStream_t)stream);
}

kfbi_status kfbi_plan_set_geometry(kfbi_plan *p, const kfbi_geometry *g) {
  KFBI_TRY(check_plan(p));
  if (!g) return fail(KFBI_E_CONFIG, "null geometry");
  if (g->n_ctl < 8) return fail(KFBI_E_CONFIG, "control point count must be >= 8");
  const int m = p->m;
  p->n_ctl = g->n_ctl;
  p->n_edges = g->n_edges;
  p->n_rec = g->n_rec;
  p->n_groups = g->n_groups;
  p->w_ld = (g->n_ctl + 1) & ~1;
  const int n = g->n_ctl;
  cudaError_t e = cudaSuccess;
#define UP(buf, ptr, cnt) \
  if (e == cudaSuccess) e = upload(p->buf, ptr, (size_t)(cnt))
  p->W.release();
  p->w_ready = p->w_explicit = false;
  p->spec_ok = false;
  if (g->edge_theta && g->ctl_theta) {
    UP(edge_theta_d, g->edge_theta, g->n_edges > 0 ? g->n_edges : 1);
    UP(ctl_theta_d, g->ctl_theta, n);
    // the spectral form needs the reference's controls theta_j = 2 pi j / n
    // (geometry.py:393, same operation order) and the trig branch (even n >= 32)
    bool eq = (n % 2) == 0 && n >= 32;
    for (int j = 0; eq && j < n; ++j) eq = g->ctl_theta[j] == 2.0 * 3.141592653589793 * j / n;
    p->spec_ok = eq;
    // edge groups of one axis for the spectral kernels: axis-0 edges, then
    // axis-1 edges, each class padded to a multiple of 4 with -1
    std::vector<int> perm;
    for (int ax = 0; ax < 2; ++ax) {
      for (int ed = 0; ed < g->n_edges; ++ed)
        if ((g->edge_axis[ed] != 0) == (ax == 1)) perm.push_back(ed);
      while (perm.size() % 4) perm.push_back(-1);
    }
    if (perm.empty()) perm.assign(4, -1);
    p->n_perm = (int)perm.size();
    UP(edge_perm, perm.data(), perm.size());
  }
  if (g->w_edges) {
    std::vector<double> wpad((size_t)g->n_edges * p->w_ld, 0.0);
    for (int ed = 0; ed < g->n_edges; ++ed)
      std::memcpy(&wpad[(size_t)ed * p->w_ld], g->w_edges + (size_t)ed * n, n * sizeof(double));
    UP(W, wpad.data(), wpad.size());
    p->w_ready = p->w_explicit = true;
  } else if (!g->edge_theta || !g->ctl_theta || (n % 2) != 0 || n < 32) {
    return fail(KFBI_E_CONFIG, "device W build needs edge_theta / ctl_theta and an even n_ctl >= 32");
  }
  UP(edge_axis, reinterpret_cast<const signed char *>(g->edge_axis), g->n_edges);
  UP(rec_edge, g->rec_edge, g->n_rec);
  UP(rec_d, g->rec_d, g->n_rec);
  UP(rec_sigma, g->rec_sigma, g->n_rec);
  UP(group_start, g->group_start, g->n_groups + 1);
  UP(group_node, g->group_node, g->n_groups);
  UP(row_group, g->row_group, m + 2);
  UP(deriv_col, g->deriv_col, n);
  UP(speed, g->speed, n);
  UP(tangent, g->tangent, 2 * n);
  UP(normal, g->normal, 2 * n);
  UP(dtan_ds, g->dtan_ds, 2 * n);
  UP(inv3, g->inv3, 9 * n);
  UP(stencil, g->stencil, 6 * n);
  UP(ainv_rows, g->ainv_rows, 18 * n);
  UP(jcoef, g->jcoef, 36 * n);
#undef UP
  // unique six-point stencil nodes grouped by row (trace-only sweep 1)
  if (e == cudaSuccess) {
    std::vector<std::pair<int, int>> nodes;       // (flat node, entry)
    nodes.reserve(6 * (size_t)n);
    for (int q = 0; q < 6 * n; ++q) nodes.emplace_back(g->stencil[q], q);
    std::sort(nodes.begin(), nodes.end());
    // grouped by row PAIR (2q, 2q+1); node code = 2 column + (row & 1)
    std::vector<int> rows, rowptr, cols, map(6 * (size_t)n);
    int last = -1, uniq = -1, lastpair = -1;
    for (const auto &pr : nodes) {
      if (pr.first != last) {
        last = pr.first;
        ++uniq;
        const int j = pr.first / (m + 1), i = pr.first - j * (m + 1);
        if ((j >> 1) != lastpair) {
          rows.push_back(j >> 1);
          rowptr.push_back(uniq);
          lastpair = j >> 1;
        }
        cols.push_back(2 * i + (j & 1));
      }
      map[pr.second] = uniq;
    }
    rowptr.push_back(uniq + 1);
    p->sn_nrows = (int)rows.size();
    p->sn_nodes = uniq + 1;
    if ((e = upload(p->sn_rows, rows.data(), rows.size())) == cudaSuccess &&
        (e = upload(p->sn_rowptr, rowptr.data(), rowptr.size())) == cudaSuccess &&
        (e = upload(p->sn_cols, cols.data(), cols.size())) == cudaSuccess &&
        (e = upload(p->sn_map, map.data(), map.size())) == cudaSuccess &&
        (e = p->sn_vals.ensure((size_t)p->sn_nodes)) == cudaSuccess)
      e = p->sn_v13.ensure(13 * (size_t)n);
  }
  // odd grid rows x 16-element chunks holding six-point stencil nodes: the
  // trace-only first sweep solves only these chunks of the FACR odd rows
  // (rows_odd_facr_sparse); every chunk's 32-element windows must stay
  // clear of x = 0 and x = M (the chunk never needs the x = 0 boundary term)
  if (e == cudaSuccess) {
    std::vector<long long> keys;
    bool ok = m >= 512;
    for (int q = 0; q < 6 * n && ok; ++q) {
      const int node = g->stencil[q];
      const int j = node / (m + 1), i = node - j * (m + 1);
      if (!(j & 1)) continue;
      const int ch = i / 16, s0 = 16 * ch;
      if (s0 < 64 || s0 + 16 + 32 > m - 1) ok = false;   // windows of ODD_W = 32
      keys.push_back((long long)j * (m / 16 + 1) + ch);
    }
    p->n_oc = 0;
    if (ok && !keys.empty()) {
      std::sort(keys.begin(), keys.end());
      keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
      std::vector<int2> lst;
      lst.reserve(keys.size());
      for (long long k : keys) lst.push_back(make_int2((int)(k / (m / 16 + 1)), (int)(k % (m / 16 + 1))));
      if ((e = upload(p->oc_list, lst.data(), lst.size())) == cudaSuccess) p->n_oc = (int)lst.size();
      // even rows a trace sweep reads: stencil rows and the neighbours of
      // the odd stencil rows (their windows)
      std::vector<unsigned char> need((size_t)m / 2 + 1, 0);
      for (int q = 0; q < 6 * n; ++q) {
        const int j = g->stencil[q] / (m + 1);
        if (j & 1) {
          need[(size_t)(j - 1) / 2] = 1;
          need[(size_t)(j + 1) / 2] = 1;
        } else {
          need[(size_t)j / 2] = 1;
        }
      }
      if (e == cudaSuccess) e = upload(p->need_trace, need.data(), need.size());
      size_t cnt = 0;
      for (unsigned char c : need) cnt += c;
      p->frac[0] = (double)cnt / (double)need.size();
      p->frac[2] = (double)lst.size() / ((double)(m / 2) * (m / 16));
    }
  }
  if (e == cudaSuccess) e = p->gsum.ensure((size_t)(g->n_groups > 0 ? g->n_groups : 1));
  if (e == cudaSuccess) e = p->d1.ensure(n);
  if (e == cudaSuccess) e = p->psi_s.ensure(n);
  if (e == cudaSuccess) e = p->jm.ensure(6 * (size_t)n);
  if (e == cudaSuccess) e = p->jv.ensure(3 * (size_t)(g->n_edges > 0 ? g->n_edges : 1));
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("geometry upload: ") + cudaGetErrorString(e));
  p->has_geo = true;
  p->op_valid = false;
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_interp(kfbi_plan *p, int32_t mode) {
  KFBI_TRY(check_plan(p));
  if (mode < 0 || mode > 2) return fail(KFBI_E_CONFIG, "interp mode: 0 auto, 1 W rows, 2 spectral");
  if (mode == 2 && p->has_geo && (!p->spec_ok || p->w_explicit))
    return fail(KFBI_E_CONFIG, "spectral edge values need the reference's equispaced controls and even n >= 32");
  p->interp_mode = mode;
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_colsolver(kfbi_plan *p, int32_t mode) {
  KFBI_TRY(check_plan(p));
  if (mode < 0 || mode > 2) return fail(KFBI_E_CONFIG, "column solver: 0 auto, 1 tridiagonal, 2 DST-I");
  if (p->col_mode != mode) p->op_valid = false;   // the trace operator follows the solver
  p->col_mode = mode;
  return KFBI_OK;
}

kfbi_status kfbi_plan_get_colsolver(kfbi_plan *p, int32_t *mode) {
  KFBI_TRY(check_plan(p));
  if (!mode) return fail(KFBI_E_CONFIG, "null argument");
  *mode = p->col_mode;
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_facr(kfbi_plan *p, int32_t on) {
  KFBI_TRY(check_plan(p));
  if (p->facr != (on != 0)) p->op_valid = false;   // the trace operator follows the solver
  p->facr = on != 0;
  return KFBI_OK;
}

kfbi_status kfbi_plan_facr_for(kfbi_plan *p, double kre, double kim, int32_t *on) {
  KFBI_TRY(check_plan(p));
  if (!on) return fail(KFBI_E_CONFIG, "null argument");
  *on = (p->facr && col_use_tri(p, kre, kim) && p->m >= 64 &&
         (p->m <= 8192 || (kim == 0.0 && p->m == 16384))) ? 1 : 0;
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_trace_sweep(kfbi_plan *p, int32_t on) {
  KFBI_TRY(check_plan(p));
  p->trace_sweep = on != 0;
  return KFBI_OK;
}

kfbi_status kfbi_plan_colsolver_for(kfbi_plan *p, double kre, double kim, int32_t *tridiagonal,
                                    double *bound) {
  KFBI_TRY(check_plan(p));
  if (tridiagonal) *tridiagonal = col_use_tri(p, kre, kim) ? 1 : 0;
  if (bound) *bound = col_deviation_bound(p, kre, kim);
  return KFBI_OK;
}

kfbi_status kfbi_plan_get_interp(kfbi_plan *p, int32_t *spectral) {
  KFBI_TRY(check_geo(p));
  if (!spectral) return fail(KFBI_E_CONFIG, "null argument");
  *spectral = use_spectral(p) ? 1 : 0;
  return KFBI_OK;
}

kfbi_status kfbi_plan_copy_w(kfbi_plan *p, int32_t row0, int32_t nrows, double *out) {
  KFBI_TRY(check_geo(p));
  KFBI_TRY(ensure_w(p));
  if (!out || row0 < 0 || nrows < 0 || row0 + nrows > p->n_edges)
    return fail(KFBI_E_CONFIG, "copy_w: bad row range");
  cudaError_t e = cudaMemcpy2D(out, (size_t)p->n_ctl * sizeof(double), p->W.p + (size_t)row0 * p->w_ld,
                               (size_t)p->w_ld * sizeof(double), (size_t)p->n_ctl * sizeof(double),
                               (size_t)nrows, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("copy_w: ") + cudaGetErrorString(e));
  return KFBI_OK;
}

kfbi_status kfbi_jumps(kfbi_plan *p, int32_t dtype, double kre, double kim, const void *phi,
                       const void *psi, const void *fg, double fg_sign, void *jm, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KFBI_C128) return jumps_T<double2>(p, kre, kim, phi, psi, fg, fg_sign, jm, nullptr, s);
  if (kim != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  return jumps_T<double>(p, kre, kim, phi, psi, fg, fg_sign, jm, nullptr, s);
}

kfbi_status kfbi_corrections(kfbi_plan *p, int32_t dtype, const void *jm, void *c, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  const bool cplx = dtype == KFBI_C128;
  if (cplx) KFBI_TRY(edges_T<double2>(p, jm, p->jv.p, nullptr, s));
  else KFBI_TRY(edges_T<double>(p, jm, p->jv.p, nullptr, s));
  // scatter group sums into a zeroed full grid
  const size_t es = cplx ? sizeof(double2) : sizeof(double);
  KFBI_CUDA(cudaMemsetAsync(c, 0, (size_t)(p->m + 1) * (p->m + 1) * es, s), "jumps-and-corrections");
  if (p->n_groups == 0) return KFBI_OK;
  const int blocks = (p->n_groups + 255) / 256;
  if (cplx) {
    CorrArgs<double2> ca = corr_args<double2>(p, reinterpret_cast<const double2 *>(p->jv.p));
    return launch(p, KFBI_K_JUMPS, s, [&] {
      scatter_groups_kernel<double2><<<blocks, 256, 0, s>>>(ca, p->n_groups, static_cast<double2 *>(c));
    });
  }
  CorrArgs<double> ca = corr_args<double>(p, reinterpret_cast<const double *>(p->jv.p));
  return launch(p, KFBI_K_JUMPS, s, [&] {
    scatter_groups_kernel<double><<<blocks, 256, 0, s>>>(ca, p->n_groups, static_cast<double *>(c));
  });
}

kfbi_status kfbi_interface_solve(kfbi_plan *p, int32_t dtype, double kre, double kim, const void *F,
                                 const void *jm, void *u, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KFBI_C128) KFBI_TRY(edges_T<double2>(p, jm, p->jv.p, nullptr, s));
  else KFBI_TRY(edges_T<double>(p, jm, p->jv.p, nullptr, s));
  return box_dispatch(p, dtype, kre, kim, F, 1.0, p->jv.p, u, nullptr, s);
}

kfbi_status kfbi_extract(kfbi_plan *p, int32_t dtype, const void *u, const void *jm, void *out,
                         void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  ExtractArgs x = extract_args(p);
  const int blocks = (p->n_ctl + 255) / 256;
  if (dtype == KFBI_C128)
    return launch(p, KFBI_K_EXTRACT, s, [&] {
      extract_kernel<double2><<<blocks, 256, 0, s>>>(x, static_cast<const double2 *>(u),
                                                     static_cast<const double2 *>(jm),
                                                     static_cast<double2 *>(out));
    });
  return launch(p, KFBI_K_EXTRACT, s, [&] {
    extract_kernel<double><<<blocks, 256, 0, s>>>(x, static_cast<const double *>(u),
                                                  static_cast<const double *>(jm),
                                                  static_cast<double *>(out));
  });
}

kfbi_status kfbi_classify_nodes(int32_t device, int32_t kind, const double *params, const double *x,
                                const double *y, int32_t m, double tol, uint8_t *interior,
                                int32_t *n_ambiguous, int64_t *ambiguous, int32_t cap) {
  if (!params || !x || !y || !interior || !n_ambiguous || m < 1 || cap < 0)
    return fail(KFBI_E_CONFIG, "classify: null argument");
  if (kind < 0 || kind > 2) return fail(KFBI_E_CONFIG, "classify: curve kind 0 circle, 1 ellipse, 2 star");
  KFBI_CUDA(cudaSetDevice(device), "classify-nodes");
  CurveDesc c;
  c.kind = kind;
  c.cx = params[0];
  c.cy = params[1];
  c.p0 = params[2];
  c.p1 = kind >= 1 ? params[3] : 0.0;
  c.p2 = kind == 2 ? params[4] : 0.0;
  const size_t n1 = (size_t)m + 1, total = n1 * n1;
  double *dx = nullptr, *dy = nullptr;
  unsigned char *dint = nullptr;
  int *dn = nullptr;
  long long *damb = nullptr;
  cudaError_t e = cudaMalloc(&dx, n1 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dy, n1 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dint, total);
  if (e == cudaSuccess) e = cudaMalloc(&dn, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&damb, (size_t)(cap > 0 ? cap : 1) * sizeof(long long));
  if (e == cudaSuccess) e = cudaMemcpy(dx, x, n1 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dy, y, n1 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dn, 0, sizeof(int));
  if (e == cudaSuccess) {
    const double band = kind == 2 ? 1e-12 : 0.0;    // polynomials are exact
    classify_kernel<<<148 * 8, 256>>>(c, dx, dy, m, tol, band, dint, dn, damb, cap);
    e = cudaGetLastError();
  }
  int nh = 0;
  if (e == cudaSuccess) e = cudaMemcpy(interior, dint, total, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&nh, dn, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && nh > 0 && cap > 0)
    e = cudaMemcpy(ambiguous, damb, (size_t)(nh < cap ? nh : cap) * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(dint);
  cudaFree(dn);
  cudaFree(damb);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("kernel 'classify-nodes': ") + cudaGetErrorString(e));
  *n_ambiguous = nh;
  return KFBI_OK;
}

kfbi_status kfbi_gmres(kfbi_plan *p, const kfbi_bvp *b, int32_t restart, kfbi_bvp_result *res,
                       void *stream) {
  KFBI_TRY(check_geo(p));
  if (!b || !res) return fail(KFBI_E_CONFIG, "null argument");
  if (b->max_iter < 1) return fail(KFBI_E_CONFIG, "max iterations must be >= 1");
  if (!(b->gamma > 0.0 && b->gamma < 1.0)) return fail(KFBI_E_CONFIG, "gamma must lie in (0,1)");
  if (!(b->tol > 0.0)) return fail(KFBI_E_CONFIG, "tolerance must be positive");
  if (restart < 1 || restart > 64) return fail(KFBI_E_CONFIG, "GMRES restart must lie in 1..64");
  const bool cplx = b->dtype == KFBI_C128;
  if (!cplx && b->kappa_im != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  if (b->bc_kind != 0 && b->bc_kind != 1) return fail(KFBI_E_CONFIG, "unknown boundary condition kind");
  if (b->bc_kind == 1 && !p->has_os)
    return fail(KFBI_E_CONFIG, "Neumann BVP: one-sided extraction tables missing (kfbi_plan_set_onesided)");
  if (b->use_operator &&
      (!p->op_valid || p->op_dtype != b->dtype || p->op_kre != b->kappa_re || p->op_kim != b->kappa_im ||
       p->op_bc != b->bc_kind * 2 + b->box_bc))
    return fail(KFBI_E_CONFIG, "trace operator not built for this kappa / dtype (kfbi_build_trace_operator)");
  cudaError_t e = p->history.ensure(b->max_iter);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, "history allocation failed");
  cudaStream_t s = (cudaStream_t)stream;
  if (cplx) return gmres_T<double2>(p, b, restart, res, s);
  return gmres_T<double>(p, b, restart, res, s);
}

kfbi_status kfbi_richardson(kfbi_plan *p, const kfbi_bvp *b, kfbi_bvp_result *res, void *stream) {
  KFBI_TRY(check_geo(p));
  if (!b || !res) return fail(KFBI_E_CONFIG, "null argument");
  if (b->max_iter < 1) return fail(KFBI_E_CONFIG, "max iterations must be >= 1");
  if (!(b->gamma > 0.0 && b->gamma < 1.0)) return fail(KFBI_E_CONFIG, "gamma must lie in (0,1)");
  if (!(b->tol > 0.0)) return fail(KFBI_E_CONFIG, "tolerance must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  const bool cplx = b->dtype == KFBI_C128;
  if (!cplx && b->kappa_im != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  cudaError_t e = p->history.ensure(b->max_iter);
  if (e != cudaSuccess) return fail(KFBI_E_CUDA, "history allocation failed");
  if (b->bc_kind != 0 && b->bc_kind != 1) return fail(KFBI_E_CONFIG, "unknown boundary condition kind");
  if (b->box_bc != KFBI_DIRICHLET_ZERO && b->box_bc != KFBI_NEUMANN_ZERO)
    return fail(KFBI_E_CONFIG, "unknown box boundary condition");
  if (b->bc_kind == 1 && !p->has_os)
    return fail(KFBI_E_CONFIG, "Neumann BVP: one-sided extraction tables missing (kfbi_plan_set_onesided)");
  const bool use_op = b->use_operator != 0;
  bool sync_trace_only = false;
  const size_t es = cplx ? sizeof(double2) : sizeof(double);
  if (use_op) {
    if (!p->op_valid || p->op_dtype != b->dtype || p->op_kre != b->kappa_re || p->op_kim != b->kappa_im ||
        p->op_bc != b->bc_kind * 2 + b->box_bc)
      return fail(KFBI_E_CONFIG, "trace operator not built for this kappa / dtype (kfbi_build_trace_operator)");
    KFBI_TRY(ensure_op_scratch(p));
  }
  KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] { rich_init_kernel<<<1, 1, 0, s>>>(p->st.p, b->max_iter, b->tol); }));
  if (use_op)
    KFBI_CUDA(cudaMemcpyAsync(p->phi0.p, b->density, p->n_ctl * es, cudaMemcpyDeviceToDevice, s),
              "density-update");
  if (use_op && b->log_slot >= 0) {
    // asynchronous operator form: no host sync at all; the device decides
    // whether the full pipeline must recompute the field and logs the step
    if (b->log_slot >= p->log_cap) return fail(KFBI_E_CONFIG, "log slot out of range (kfbi_log_reserve)");
    KFBI_TRY(ensure_async_scratch(p));
    const bool ft = facr_trace_ok(p, b);
    const bool tr = ft || trace_sweep_ok(p, b);
    if (ft && cplx) KFBI_TRY(sweep1_facr_trace<double2>(p, b, s));
    else if (ft) KFBI_TRY(sweep1_facr_trace<double>(p, b, s));
    else if (tr && cplx) KFBI_TRY(sweep1_trace<double2>(p, b, s));
    else if (tr) KFBI_TRY(sweep1_trace<double>(p, b, s));
    else if (cplx) KFBI_TRY(sweep<double2>(p, b, s));
    else KFBI_TRY(sweep<double>(p, b, s));
    KFBI_CUDA(cudaMemcpyAsync(p->trace1.p, b->bc_kind ? b->trace_un : b->trace_u, p->n_ctl * es, cudaMemcpyDeviceToDevice, s),
              "density-update");
    if (b->max_iter > 1) {
      if (cplx) KFBI_TRY(op_solve<double2>(p, b, s));
      else KFBI_TRY(op_solve<double>(p, b, s));
    }
    StepLog *entry = p->log.p + b->log_slot;
    int *skip = p->skip.p;
    if (cplx) {
      KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
        op_finalize_kernel<double2><<<(p->n_ctl + 255) / 256, 256, 0, s>>>(p->st.p, p->n_ctl, static_cast<double2 *>(b->density),
                                                      p->phi_prev.p, p->phik1.p, skip, entry,
                                                      tr ? p->phi0.p : nullptr);
      }));
      KFBI_TRY(final_pipeline<double2>(p, b, p->phik1.p, s, skip));
    } else {
      KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
        op_finalize_kernel<double><<<(p->n_ctl + 255) / 256, 256, 0, s>>>(
            p->st.p, p->n_ctl, static_cast<double *>(b->density),
            reinterpret_cast<const double *>(p->phi_prev.p), reinterpret_cast<double *>(p->phik1.p),
            skip, entry, tr ? reinterpret_cast<const double *>(p->phi0.p) : nullptr);
      }));
      KFBI_TRY(final_pipeline<double>(p, b, p->phik1.p, s, skip));
    }
    res->iterations = -1;     // pending: read with kfbi_log_fetch
    res->converged = -1;
    res->residual = 0.0;
    return KFBI_OK;
  }
  if (use_op) {
    // sweep 1 through the pipeline, then every further sweep inside one
    // cooperative launch; a single host sync per solve
    const bool ft = facr_trace_ok(p, b);
    const bool tr = ft || trace_sweep_ok(p, b);
    if (ft && cplx) KFBI_TRY(sweep1_facr_trace<double2>(p, b, s));
    else if (ft) KFBI_TRY(sweep1_facr_trace<double>(p, b, s));
    else if (tr && cplx) KFBI_TRY(sweep1_trace<double2>(p, b, s));
    else if (tr) KFBI_TRY(sweep1_trace<double>(p, b, s));
    else if (cplx) KFBI_TRY(sweep<double2>(p, b, s));
    else KFBI_TRY(sweep<double>(p, b, s));
    sync_trace_only = tr;
    KFBI_CUDA(cudaMemcpyAsync(p->trace1.p, b->bc_kind ? b->trace_un : b->trace_u, p->n_ctl * es, cudaMemcpyDeviceToDevice, s),
              "density-update");
    if (b->max_iter > 1) {
      if (cplx) KFBI_TRY(op_solve<double2>(p, b, s));
      else KFBI_TRY(op_solve<double>(p, b, s));
    }
    KFBI_CUDA(cudaMemcpyAsync(p->st_host, p->st.p, sizeof(RichState), cudaMemcpyDeviceToHost, s),
              "density-update");
    KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
  } else {
    // trace-only sweeps (FACR with the stencil chunks of the odd rows): each
    // sweep keeps the density it started from, the field comes from one full
    // pipeline after the loop
    const bool ft = facr_trace_ok(p, b);
    if (ft) KFBI_TRY(ensure_op_scratch(p));
    int enqueued = 0;
    int batch = b->sweeps_hint > 0 ? b->sweeps_hint : 4;
    for (;;) {
      int nb = batch;
      if (nb > b->max_iter - enqueued) nb = b->max_iter - enqueued;
      for (int k = 0; k < nb; ++k) {
        if (ft) {
          KFBI_TRY(launch(p, KFBI_K_DENSITY, s, [&] {
            if (cplx)
              copy_running_kernel<double2><<<64, 256, 0, s>>>(p->st.p, p->n_ctl,
                                                             static_cast<const double2 *>(b->density),
                                                             p->phi_prev.p);
            else
              copy_running_kernel<double><<<64, 256, 0, s>>>(p->st.p, p->n_ctl,
                                                            static_cast<const double *>(b->density),
                                                            reinterpret_cast<double *>(p->phi_prev.p));
          }));
          if (cplx) KFBI_TRY(sweep1_facr_trace<double2>(p, b, s));
          else KFBI_TRY(sweep1_facr_trace<double>(p, b, s));
          continue;
        }
        if (cplx) KFBI_TRY(sweep<double2>(p, b, s));
        else KFBI_TRY(sweep<double>(p, b, s));
      }
      enqueued += nb;
      KFBI_CUDA(cudaMemcpyAsync(p->st_host, p->st.p, sizeof(RichState), cudaMemcpyDeviceToHost, s),
                "density-update");
      KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
      if (p->st_host->done != 0 || enqueued >= b->max_iter) break;
      batch = 2;
    }
    if (ft) {
      // the field and traces of the last sweep, from the density it started from
      if (cplx) KFBI_TRY(final_pipeline<double2>(p, b, p->phi_prev.p, s));
      else KFBI_TRY(final_pipeline<double>(p, b, p->phi_prev.p, s));
    }
  }
  if (use_op && sync_trace_only && p->st_host->iters == 1 && p->st_host->done == 1) {
    // converged at sweep 1, whose field was not formed: recompute it from phi_0
    if (cplx) KFBI_TRY(final_pipeline<double2>(p, b, p->phi0.p, s));
    else KFBI_TRY(final_pipeline<double>(p, b, p->phi0.p, s));
  }
  if (use_op && p->st_host->iters >= 2) {
    // after K sweeps: phi_K sits in density when K is odd, in phi_prev when
    // K is even (op_sweep ping-pong); phi_(K-1) in the other buffer
    const int K = p->st_host->iters;
    void *phiK = (K & 1) ? b->density : (void *)p->phi_prev.p;
    void *phiK1 = (K & 1) ? (void *)p->phi_prev.p : b->density;
    if (p->st_host->done == 1) {
      if (cplx) KFBI_TRY(final_pipeline<double2>(p, b, phiK1, s));
      else KFBI_TRY(final_pipeline<double>(p, b, phiK1, s));
    }
    if (phiK != b->density)
      KFBI_CUDA(cudaMemcpyAsync(b->density, phiK, p->n_ctl * es, cudaMemcpyDeviceToDevice, s),
                "density-update");
  }
  const RichState &h = *p->st_host;
  res->iterations = h.iters;
  res->converged = h.done == 1;
  res->residual = h.last_res;
  if (res->history && h.iters > 0)
    KFBI_CUDA(cudaMemcpy(res->history, p->history.p, sizeof(double) * h.iters, cudaMemcpyDeviceToHost),
              "density-update");
  if (h.done != 1) {
    char msg[256];
    std::snprintf(msg, sizeof msg,
                  "Richardson iteration did not reach tol=%g within %d sweeps (last density update %.3e)",
                  b->tol, b->max_iter, h.last_res);
    return fail(KFBI_E_NOCONV, msg);
  }
  return KFBI_OK;
}

kfbi_status kfbi_build_trace_operator_bc(kfbi_plan *p, int32_t dtype, int32_t bc_kind, int32_t box_bc,
                                         double kre, double kim, void *stream) {
  KFBI_TRY(check_geo(p));
  if (bc_kind == 1 && !p->has_os)
    return fail(KFBI_E_CONFIG, "Neumann operator: one-sided extraction tables missing");
  cudaStream_t s = (cudaStream_t)stream;
  if (p->n_ctl > op_max_ctl(p))
    return fail(KFBI_E_CONFIG, "operator form: n_ctl = " + std::to_string(p->n_ctl) + " exceeds " +
                                   std::to_string(op_max_ctl(p)) + " (32 rows per SM); use the pipeline form");
  if (dtype == KFBI_C128) return build_operator_T<double2>(p, kre, kim, bc_kind, box_bc, s);
  if (kim != 0.0) return fail(KFBI_E_CONFIG, "complex kappa requires the c128 path");
  return build_operator_T<double>(p, kre, kim, bc_kind, box_bc, s);
}

kfbi_status kfbi_operator_max_controls(kfbi_plan *p, int32_t *n_max) {
  KFBI_TRY(check_plan(p));
  if (!n_max) return fail(KFBI_E_CONFIG, "null argument");
  *n_max = op_max_ctl(p);
  return KFBI_OK;
}

kfbi_status kfbi_build_trace_operator(kfbi_plan *p, int32_t dtype, double kre, double kim, void *stream) {
  return kfbi_build_trace_operator_bc(p, dtype, 0, KFBI_DIRICHLET_ZERO, kre, kim, stream);
}

kfbi_status kfbi_box_solve_bc(kfbi_plan *p, int32_t dtype, int32_t box_bc, double kre, double kim,
                              const void *rhs, void *u, void *stream) {
  KFBI_TRY(check_plan(p));
  if (!rhs || !u) return fail(KFBI_E_CONFIG, "null field pointer");
  return box_dispatch(p, dtype, kre, kim, rhs, 1.0, nullptr, u, nullptr, (cudaStream_t)stream, box_bc);
}

kfbi_status kfbi_interface_solve_bc(kfbi_plan *p, int32_t dtype, int32_t box_bc, double kre, double kim,
                                    const void *F, const void *jm, void *u, void *stream) {
  KFBI_TRY(check_geo(p));
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == KFBI_C128) KFBI_TRY(edges_T<double2>(p, jm, p->jv.p, nullptr, s));
  else KFBI_TRY(edges_T<double>(p, jm, p->jv.p, nullptr, s));
  return box_dispatch(p, dtype, kre, kim, F, 1.0, p->jv.p, u, nullptr, s, box_bc);
}

kfbi_status kfbi_plan_set_onesided(kfbi_plan *p, int32_t n_ctl, const int32_t *stencil7,
                                   const double *rows, const uint8_t *fallback) {
  KFBI_TRY(check_geo(p));
  if (n_ctl != p->n_ctl || !stencil7 || !rows || !fallback)
    return fail(KFBI_E_CONFIG, "one-sided tables: bad argument");
  cudaError_t e;
  if ((e = upload(p->os_stencil, stencil7, (size_t)7 * n_ctl)) != cudaSuccess ||
      (e = upload(p->os_rows, rows, (size_t)21 * n_ctl)) != cudaSuccess ||
      (e = upload(p->os_fb, fallback, (size_t)n_ctl)) != cudaSuccess)
    return fail(KFBI_E_CUDA, std::string("one-sided tables: ") + cudaGetErrorString(e));
  p->has_os = true;
  return KFBI_OK;
}

kfbi_status kfbi_extract_onesided(kfbi_plan *p, int32_t dtype, const void *u, const void *jm, void *out,
                                  void *stream) {
  KFBI_TRY(check_geo(p));
  if (!p->has_os) return fail(KFBI_E_CONFIG, "one-sided extraction tables missing");
  cudaStream_t s = (cudaStream_t)stream;
  ExtractArgs x = extract_args(p, true);
  const int blocks = (p->n_ctl + 255) / 256;
  if (dtype == KFBI_C128)
    return launch(p, KFBI_K_EXTRACT, s, [&] {
      extract_kernel<double2><<<blocks, 256, 0, s>>>(x, static_cast<const double2 *>(u),
                                                     static_cast<const double2 *>(jm),
                                                     static_cast<double2 *>(out));
    });
  return launch(p, KFBI_K_EXTRACT, s, [&] {
    extract_kernel<double><<<blocks, 256, 0, s>>>(x, static_cast<const double *>(u),
                                                  static_cast<const double *>(jm),
                                                  static_cast<double *>(out));
  });
}

kfbi_status kfbi_log_reserve(kfbi_plan *p, int32_t count) {
  KFBI_TRY(check_plan(p));
  if (count <= p->log_cap) return KFBI_OK;
  DevBuf<StepLog> nb;
  cudaError_t e = nb.ensure((size_t)count);
  if (e == cudaSuccess && p->log_cap > 0)
    e = cudaMemcpy(nb.p, p->log.p, sizeof(StepLog) * p->log_cap, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess) e = cudaMemset(nb.p + p->log_cap, 0, sizeof(StepLog) * (count - p->log_cap));
  if (e != cudaSuccess) {
    nb.release();
    return fail(KFBI_E_CUDA, std::string("log allocation: ") + cudaGetErrorString(e));
  }
  p->log.release();
  p->log = nb;
  nb.p = nullptr;
  p->log_cap = count;
  return KFBI_OK;
}

kfbi_status kfbi_log_norm(kfbi_plan *p, int32_t slot, int32_t which, void *stream) {
  KFBI_TRY(check_plan(p));
  if (slot < 0 || slot >= p->log_cap) return fail(KFBI_E_CONFIG, "log slot out of range");
  cudaStream_t s = (cudaStream_t)stream;
  return launch(p, KFBI_K_RHS, s, [&] { log_norm_kernel<<<1, 1, 0, s>>>(p->red.p, p->log.p + slot, which); });
}

kfbi_status kfbi_log_fetch(kfbi_plan *p, int32_t first, int32_t count, kfbi_step_log *out,
                           void *stream) {
  KFBI_TRY(check_plan(p));
  if (first < 0 || count < 0 || first + count > p->log_cap)
    return fail(KFBI_E_CONFIG, "log range out of bounds");
  static_assert(sizeof(kfbi_step_log) == sizeof(StepLog), "log layout");
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemcpyAsync(out, p->log.p + first, sizeof(StepLog) * count, cudaMemcpyDeviceToHost, s),
            "density-update");
  KFBI_CUDA(cudaStreamSynchronize(s), "density-update");
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_exterior_zero(kfbi_plan *p, int32_t on) {
  KFBI_TRY(check_plan(p));
  p->ext_zero = on != 0;
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_field_chunks(kfbi_plan *p, const int32_t *pairs, int64_t count) {
  KFBI_TRY(check_plan(p));
  if (count < 0 || (count > 0 && !pairs)) return fail(KFBI_E_CONFIG, "field chunks: bad arguments");
  const int nch = p->m / 16;
  for (int64_t q = 0; q < count; ++q) {
    const int j = pairs[2 * q], ch = pairs[2 * q + 1], s0 = 16 * ch;
    if (j < 1 || j > p->m - 1 || !(j & 1) || ch < 0 || ch >= nch || s0 < 64 || s0 + 16 + 32 > p->m - 1)
      return fail(KFBI_E_CONFIG, "field chunks: (odd row, chunk) pairs with windows inside the box");
  }
  p->n_fc = 0;
  if (count > 0) {
    // per odd row the covering chunk range (the odd-row pass keeps its
    // thread-per-chunk layout and skips the rest of the row)
    std::vector<int2> span((size_t)p->m / 2, make_int2(1, 0));
    for (int64_t q = 0; q < count; ++q) {
      int2 &sp = span[(size_t)(pairs[2 * q] - 1) / 2];
      const int ch = pairs[2 * q + 1];
      if (sp.x > sp.y) sp = make_int2(ch, ch);
      else sp = make_int2(std::min(sp.x, ch), std::max(sp.y, ch));
    }
    cudaError_t e = upload(p->fc_span, span.data(), span.size());
    // even rows the masked caller (or the odd rows' windows) read: between
    // the first and last odd row with chunks, one row beyond each (the
    // interior and the stencils of a closed curve occupy a contiguous band
    // of rows; an even row inside the band next to no chunk row still holds
    // interior nodes, so the whole band is kept)
    std::vector<unsigned char> need((size_t)p->m / 2 + 1, 0);
    int jlo = p->m, jhi = -1;
    for (int64_t q = 0; q < count; ++q) {
      jlo = std::min(jlo, (int)pairs[2 * q]);
      jhi = std::max(jhi, (int)pairs[2 * q]);
    }
    for (int j = std::max(jlo - 1, 0); j <= std::min(jhi + 1, p->m); ++j)
      if (!(j & 1)) need[(size_t)j / 2] = 1;
    if (e == cudaSuccess) e = upload(p->need_field, need.data(), need.size());
    if (e != cudaSuccess) return fail(KFBI_E_CUDA, std::string("field chunks: ") + cudaGetErrorString(e));
    p->n_fc = (int)count;
    size_t cnt = 0, chunks = 0;
    for (unsigned char c : need) cnt += c;
    for (const int2 &sp : span)
      if (sp.x <= sp.y) chunks += (size_t)(sp.y - sp.x + 1);
    p->frac[1] = (double)cnt / (double)need.size();
    p->frac[3] = (double)chunks / ((double)(p->m / 2) * (p->m / 16));
  }
  return KFBI_OK;
}

kfbi_status kfbi_plan_work_fractions(kfbi_plan *p, double *out) {
  KFBI_TRY(check_plan(p));
  if (!out) return fail(KFBI_E_CONFIG, "work fractions: null output");
  for (int q = 0; q < 4; ++q) out[q] = p->frac[q];
  return KFBI_OK;
}

kfbi_status kfbi_plan_set_interior_list(kfbi_plan *p, const int32_t *idx, int64_t count) {
  KFBI_TRY(check_plan(p));
  if (count < 0 || (count > 0 && !idx)) return fail(KFBI_E_CONFIG, "interior list: bad arguments");
  p->int_idx = idx;
  p->n_int = idx ? count : 0;
  return KFBI_OK;
}

kfbi_status kfbi_log_clear(kfbi_plan *p, int32_t slot, int32_t count, void *stream) {
  KFBI_TRY(check_plan(p));
  if (slot < 0 || count < 0 || slot + count > p->log_cap) return fail(KFBI_E_CONFIG, "log range out of bounds");
  KFBI_CUDA(cudaMemsetAsync(p->log.p + slot, 0, sizeof(StepLog) * count, (cudaStream_t)stream),
            "rhs-update");
  return KFBI_OK;
}

kfbi_status kfbi_log_copy(kfbi_plan *p, int32_t src, int32_t dst, int32_t count, void *stream) {
  KFBI_TRY(check_plan(p));
  if (src < 0 || dst < 0 || count < 0 || src + count > p->log_cap || dst + count > p->log_cap)
    return fail(KFBI_E_CONFIG, "log range out of bounds");
  KFBI_CUDA(cudaMemcpyAsync(p->log.p + dst, p->log.p + src, sizeof(StepLog) * count,
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "rhs-update");
  return KFBI_OK;
}

kfbi_status kfbi_heat_rhs(kfbi_plan *p, int64_t n, const uint8_t *mask, void *u, const void *F_old,
                          void *F_new, double a, double *norm_out, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemsetAsync(p->red.p, 0, sizeof(unsigned long long), s), "rhs-update");
  KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
    auto *uu = static_cast<double *>(u);
    auto *fo = static_cast<const double *>(F_old);
    auto *fn = static_cast<double *>(F_new);
    if (aligned16({uu, fo, fn}) && !((uintptr_t)mask & 1))
      heat_rhs_kernel<true><<<pair_blocks(n), 256, 0, s>>>(n, mask, uu, fo, fn, a, p->red.p, p->ext_zero);
    else
      heat_rhs_kernel<false><<<elem_blocks(n), 256, 0, s>>>(n, mask, uu, fo, fn, a, p->red.p, p->ext_zero);
  }));
  return norm_out ? read_norm(p, s, norm_out) : KFBI_OK;
}

kfbi_status kfbi_wave_rhs(kfbi_plan *p, int64_t n, const uint8_t *mask, void *u_next,
                          const void *u_curr, const void *F_curr, const void *F_prev, void *F_new,
                          double kw, double coef, double *norm_out, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemsetAsync(p->red.p, 0, sizeof(unsigned long long), s), "rhs-update");
  KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
    auto *un = static_cast<double *>(u_next);
    auto *uc = static_cast<const double *>(u_curr);
    auto *fc = static_cast<const double *>(F_curr);
    auto *fp = static_cast<const double *>(F_prev);
    auto *fn = static_cast<double *>(F_new);
    if (aligned16({un, uc, fc, fp, fn}) && !((uintptr_t)mask & 1))
      wave_rhs_kernel<true><<<pair_blocks(n), 256, 0, s>>>(n, mask, un, uc, fc, fp, fn, kw, coef, p->red.p, p->ext_zero);
    else
      wave_rhs_kernel<false><<<elem_blocks(n), 256, 0, s>>>(n, mask, un, uc, fc, fp, fn, kw, coef, p->red.p, p->ext_zero);
  }));
  return norm_out ? read_norm(p, s, norm_out) : KFBI_OK;
}

kfbi_status kfbi_schr_ustar(kfbi_plan *p, int64_t n, int32_t mode, const void *u, const void *other,
                            double tau, void *out, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  return launch(p, KFBI_K_RHS, s, [&] {
    schr_ustar_kernel<<<elem_blocks(n), 256, 0, s>>>(n, mode, static_cast<const double2 *>(u),
                                                     static_cast<const double2 *>(other), tau,
                                                     static_cast<double2 *>(out));
  });
}

kfbi_status kfbi_nonlinear_phase(kfbi_plan *p, int64_t n, const void *ustar, const double *v,
                                 double w, double half_tau, const uint8_t *mask, void *out,
                                 double kre, double kim, void *F, double *max_res, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemsetAsync(p->red.p, 0, sizeof(unsigned long long), s), "rhs-update");
  KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
    if (mask && p->ext_zero && p->int_idx)
      nonlinear_phase_list_kernel<<<elem_blocks(p->n_int), 256, 0, s>>>(
          p->n_int, p->int_idx, static_cast<const double2 *>(ustar), nullptr, 0, 0.0, v, w, half_tau,
          static_cast<double2 *>(out), kre, kim, static_cast<double2 *>(F), p->red.p);
    else
      nonlinear_phase_kernel<<<elem_blocks(n), 256, 0, s>>>(
          n, static_cast<const double2 *>(ustar), nullptr, 0, 0.0, v, w, half_tau, mask,
          static_cast<double2 *>(out), kre, kim, static_cast<double2 *>(F), p->red.p, p->ext_zero);
  }));
  if (!max_res) return KFBI_OK;    // asynchronous: the caller logs red[0] (kfbi_log_norm)
  double r = 0.0;
  KFBI_TRY(read_norm(p, s, &r));
  if (max_res) *max_res = r;
  if (r > NEWTON_TOL || r != r) {
    char msg[160];
    std::snprintf(msg, sizeof msg, "pointwise Newton solve stalled at residual %.3e", r);
    return fail(KFBI_E_NOCONV, msg);
  }
  return KFBI_OK;
}

kfbi_status kfbi_strang_phase(kfbi_plan *p, int64_t n, int32_t mode, const void *u, const void *other,
                              double tau, const double *v, double w, double half_tau,
                              const uint8_t *mask, void *out, double kre, double kim, void *F,
                              double *max_res, void *stream) {
  KFBI_TRY(check_plan(p));
  if (!other) return fail(KFBI_E_CONFIG, "kfbi_strang_phase: `other` is required");
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemsetAsync(p->red.p, 0, sizeof(unsigned long long), s), "rhs-update");
  KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
    if (mask && p->ext_zero && p->int_idx)
      nonlinear_phase_list_kernel<<<elem_blocks(p->n_int), 256, 0, s>>>(
          p->n_int, p->int_idx, static_cast<const double2 *>(u), static_cast<const double2 *>(other),
          mode, tau, v, w, half_tau, static_cast<double2 *>(out), kre, kim, static_cast<double2 *>(F),
          p->red.p);
    else
      nonlinear_phase_kernel<<<elem_blocks(n), 256, 0, s>>>(
          n, static_cast<const double2 *>(u), static_cast<const double2 *>(other), mode, tau, v, w,
          half_tau, mask, static_cast<double2 *>(out), kre, kim, static_cast<double2 *>(F), p->red.p,
          p->ext_zero);
  }));
  if (!max_res) return KFBI_OK;
  double r = 0.0;
  KFBI_TRY(read_norm(p, s, &r));
  *max_res = r;
  if (r > NEWTON_TOL || r != r) {
    char msg[160];
    std::snprintf(msg, sizeof msg, "pointwise Newton solve stalled at residual %.3e", r);
    return fail(KFBI_E_NOCONV, msg);
  }
  return KFBI_OK;
}

kfbi_status kfbi_gather(kfbi_plan *p, int32_t dtype, int64_t n, const int32_t *idx, const void *src,
                        void *dst, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  if (n <= 0) return KFBI_OK;
  return launch(p, KFBI_K_RHS, s, [&] {
    if (dtype == KFBI_C128)
      gather_kernel<double2><<<elem_blocks(n), 256, 0, s>>>(n, idx, static_cast<const double2 *>(src),
                                                            static_cast<double2 *>(dst));
    else
      gather_kernel<double><<<elem_blocks(n), 256, 0, s>>>(n, idx, static_cast<const double *>(src),
                                                           static_cast<double *>(dst));
  });
}

kfbi_status kfbi_mask_norm(kfbi_plan *p, int32_t dtype, int64_t n, const uint8_t *mask, void *u,
                           double *norm_out, void *stream) {
  KFBI_TRY(check_plan(p));
  cudaStream_t s = (cudaStream_t)stream;
  KFBI_CUDA(cudaMemsetAsync(p->red.p, 0, sizeof(unsigned long long), s), "rhs-update");
  if (dtype == KFBI_C128)
    KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
      auto *uu = static_cast<double2 *>(u);
      if (!((uintptr_t)mask & 1))
        mask_norm_kernel<double2, true><<<pair_blocks(n), 256, 0, s>>>(n, mask, uu, p->red.p);
      else
        mask_norm_kernel<double2, false><<<elem_blocks(n), 256, 0, s>>>(n, mask, uu, p->red.p);
    }));
  else
    KFBI_TRY(launch(p, KFBI_K_RHS, s, [&] {
      auto *uu = static_cast<double *>(u);
      if (aligned16({uu}) && !((uintptr_t)mask & 1))
        mask_norm_kernel<double, true><<<pair_blocks(n), 256, 0, s>>>(n, mask, uu, p->red.p);
      else
        mask_norm_kernel<double, false><<<elem_blocks(n), 256, 0, s>>>(n, mask, uu, p->red.p);
    }));
  return norm_out ? read_norm(p, s, norm_out) : KFBI_OK;
}

kfbi_status kfbi_kernel_times(kfbi_plan *p, double *ms, int64_t *calls) {
  KFBI_TRY(check_plan(p));
  for (auto &pe : p->pending) {
    cudaEventSynchronize(pe.b);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, pe.a, pe.b) == cudaSuccess) p->ms[pe.name] += t;
    p->pool.push_back(pe.a);
    p->pool.push_back(pe.b);
  }
  p->pending.clear();
  for (int i = 0; i < KFBI_N_KERNEL_NAMES; ++i) {
    if (ms) ms[i] = p->ms[i];
    if (calls) calls[i] = p->calls[i];
  }
  return KFBI_OK;
}

kfbi_status kfbi_reset_kernel_times(kfbi_plan *p) {
  KFBI_TRY(kfbi_kernel_times(p, nullptr, nullptr));
  for (int i = 0; i < KFBI_N_KERNEL_NAMES; ++i) {
    p->ms[i] = 0.0;
    p->calls[i] = 0;
  }
  p->launches = 0;
  return KFBI_OK;
}

kfbi_status kfbi_set_timing(kfbi_plan *p, int32_t enabled) {
  KFBI_TRY(check_plan(p));
  if (!enabled) KFBI_TRY(kfbi_kernel_times(p, nullptr, nullptr));
  p->timing = enabled != 0;
  return KFBI_OK;
}

int64_t kfbi_launch_count(kfbi_plan *p) { return p ? p->launches : 0; }

}  // extern "C"
