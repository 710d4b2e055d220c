// Launch code of the box-solve passes (templates over dtype and log2 M),
// included by the per-dtype translation units box_dir_*.cu / box_neu_*.cu.
#pragma once

#include "host_common.h"
#include "box_reg.cuh"
#include "box_neu.cuh"
#include "box_real.cuh"
#include "box_tri.cuh"
#include "box_facr.cuh"

namespace kfbi {

// Launch one register-engine kernel: plain, or as clusters of Cfg::CL CTAs.
template <int LOGN, typename K, typename... Args>
cudaError_t reg_launch(K kernel, int grid, cudaStream_t s, Args... args) {
  using Cf = reg::Cfg<LOGN>;
  const size_t smem = reg::smem_bytes<LOGN>();
  if constexpr (Cf::CL == 1) {
    kernel<<<grid, Cf::CTA_T, smem, s>>>(args...);
    return cudaGetLastError();
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(Cf::CTA_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Cf::CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
  }
}

// Tridiagonal column pass (box_tri.cuh) of one (dtype, log2 M).  The
// persistent bulk-copy variant (KFBI_TRI_TMA) measured 2-9 % slower than the
// register kernel at M = 4096 (profiles/r2_v7_ab_tri.log) and is opt-in.
template <bool CPLX, int LOGN>
kfbi_status cols_tri_launch(kfbi_plan *p, const BoxArgs &a, cudaStream_t s) {
  using Tc = tri::Cfg<LOGN>;
#ifdef KFBI_TRI_TMA
  if constexpr (LOGN == tri::TMA_LOGM) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      KFBI_CUDA(cudaFuncSetAttribute(cols_tri_tma<CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tri::TMA_SMEM), "transform-cols");
    }
    const int grid = a.npl < sms ? a.npl : sms;
    return kfbi_launch(p, KFBI_K_COLS, s, [&] {
      cols_tri_tma<CPLX><<<grid, Tc::THREADS, tri::TMA_SMEM, s>>>(a);
    });
  }
#endif
  const int grid = Tc::NH == 2 ? a.npl : 2 * a.npl;
  return kfbi_launch(p, KFBI_K_COLS, s, [&] { cols_tri<CPLX, LOGN><<<grid, Tc::THREADS, 0, s>>>(a); });
}

// FACR(1) box solve (box_facr.cuh) of one (dtype, log2 M), one slab.
template <bool CPLX, int LOGN>
kfbi_status box_facr_launch(kfbi_plan *p, const BoxArgs &a0, const void *rhs, double sign,
                            const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                            void *u, cudaStream_t s) {
  if constexpr (LOGN < 6 || LOGN > 13) {
    return kfbi_fail(KFBI_E_CONFIG, "FACR box solve: 64 <= M <= 8192");
  } else {
    using Cf = reg::Cfg<LOGN>;
    using CT = typename std::conditional<CPLX, double2, double>::type;
    constexpr int M = 1 << LOGN;
    static bool attr = false;
    if (!attr) {
      const int bytes = (int)reg::smem_bytes<LOGN>();
      KFBI_CUDA(cudaFuncSetAttribute(rows_fwd_facr<CPLX, LOGN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
      KFBI_CUDA(cudaFuncSetAttribute(rows_inv_reg<CPLX, LOGN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
      attr = true;
    }
    // the group sums once (every FACR pass reads each correction several times)
    CorrArgs<CT> cc = c;
    if (c.jv && a0.gsum) {
      CT *gs = static_cast<CT *>(a0.gsum);
      KFBI_TRY(kfbi_launch(p, KFBI_K_JUMPS, s, [&] {
        group_sums_kernel<CT><<<148 * 2, 256, 0, s>>>(c, M, gs);
      }));
      cc.cval = gs;
    }
    BoxArgs a = a0;
    a.rows = M / 2;                                 // the even rows
    a.npl = CPLX ? M / 2 : M / 4;
    a.ring_end = 0;                                 // row M: written by the odd-row pass
    // zero-row flags need the one-sequence-per-CTA forward kernel
    a.rowz = (Cf::S == 1 && Cf::CL == 1) ? a0.zbuf : nullptr;

    const int nseq = CPLX ? M / 2 : M / 4;
    const int grow = Cf::CL > 1 ? nseq * Cf::CL : (nseq + Cf::S - 1) / Cf::S;
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
      return reg_launch<LOGN>(rows_fwd_facr<CPLX, LOGN>, grow, s, a, rhs, sign, cc);
    }));
    BoxArgs ar = a;
    ar.red = 1;
    KFBI_TRY((cols_tri_launch<CPLX, LOGN - 1>(p, ar, s)));
    BoxArgs ai = a;
    ai.row_step = 2;
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
      return reg_launch<LOGN>(rows_inv_reg<CPLX, LOGN>, grow, s, ai, u);
    }));
    BoxArgs ao = a0;
    ao.trow = 1;
    ao.tb_re = 1.0 + 0.5 * a0.kre * a0.h2;          // beta - 1, beta = 2 + kappa h^2 / 2
    ao.tb_im = 0.5 * a0.kim * a0.h2;
    ao.tscale = 1.0;
    using Rc = OddCfg<LOGN>;
    const int nodd = CPLX ? M / 2 : M / 4;
    constexpr size_t osm = odd_smem_bytes<LOGN>();
    static bool oattr = false;
    if (!oattr && osm > 48 * 1024) {
      KFBI_CUDA(cudaFuncSetAttribute(rows_odd_facr<CPLX, LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)osm), "diagonal-scale");
      oattr = true;
    }
    if (a0.oc_list) {                                // trace-only first sweep: the stencil chunks
      if (a0.n_oc == 0) return KFBI_OK;
      return kfbi_launch(p, KFBI_K_SCALE, s, [&] {
        rows_odd_facr_sparse<CPLX, LOGN><<<(a0.n_oc + OS_WARPS - 1) / OS_WARPS, OS_WARPS * 32, 0, s>>>(
            ao, rhs, sign, cc, u);
      });
    }
    return kfbi_launch(p, KFBI_K_SCALE, s, [&] {
      rows_odd_facr<CPLX, LOGN><<<nodd, Rc::NT, osm, s>>>(ao, rhs, sign, cc, u);
    });
  }
}

// Register-engine passes for one (dtype, log2 M); `passes` selects any of
// rows_fwd (1), cols (2), rows_inv (4).
template <bool CPLX, int LOGN>
kfbi_status box_reg_launch(kfbi_plan *p, bool tri, const BoxArgs &a, const void *rhs, double sign,
                           const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                           void *u, int passes, cudaStream_t s) {
  using Cf = reg::Cfg<LOGN>;
  static bool attr = false;   // per instantiation, process wide
  if (!attr) {
    const int bytes = (int)reg::smem_bytes<LOGN>();
    KFBI_CUDA(cudaFuncSetAttribute(rows_fwd_reg<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(rows_inv_reg<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(cols_reg<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-cols");
    attr = true;
  }
  const int nrow = CPLX ? a.rows : a.rows / 2;     // row sequences of the slab
  const int ncol = 2 * a.npl;                      // half-panel sequences
  const int grow = Cf::CL > 1 ? nrow * Cf::CL : (nrow + Cf::S - 1) / Cf::S;
  const int gcol = Cf::CL > 1 ? ncol * Cf::CL : (ncol + Cf::S - 1) / Cf::S;
  using CT = typename std::conditional<CPLX, double2, double>::type;
  if (passes & 1)
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
      return reg_launch<LOGN>(rows_fwd_reg<CPLX, LOGN>, grow, s, a, rhs, sign, CorrArgs<CT>(c));
    }));
  if ((passes & 2) && tri) KFBI_TRY((cols_tri_launch<CPLX, LOGN>(p, a, s)));
  else if (passes & 2)
    KFBI_TRY(kfbi_launch(p, KFBI_K_COLS, s, [&] { return reg_launch<LOGN>(cols_reg<CPLX, LOGN>, gcol, s, a); }));
  if (passes & 4)
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] { return reg_launch<LOGN>(rows_inv_reg<CPLX, LOGN>, grow, s, a, u); }));
  return KFBI_OK;
}

// Real data at M = 16384: one real row / column per CTA on the length-8192
// complex engine (box_real.cuh) instead of packed pairs on a two-CTA cluster.
template <int LOGN>
kfbi_status box_real_launch(kfbi_plan *p, bool tri, const BoxArgs &a, const void *rhs, double sign,
                            const CorrArgs<double> &c, void *u, int passes, cudaStream_t s) {
  constexpr int LOGL = LOGN - 1;
  static bool attr = false;
  if (!attr) {
    const int bytes = (int)reg::smem_bytes<LOGL>();
    KFBI_CUDA(cudaFuncSetAttribute(rows_fwd_real<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
              "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(rows_inv_real<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
              "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(cols_real<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
              "transform-cols");
    attr = true;
  }
  const size_t smem = reg::smem_bytes<LOGL>();
  constexpr int CT = reg::Cfg<LOGL>::CTA_T;
  if (passes & 1)
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
      rows_fwd_real<LOGN><<<a.rows, CT, smem, s>>>(a, static_cast<const double *>(rhs), sign, c);
    }));
  if ((passes & 2) && tri) KFBI_TRY((cols_tri_launch<false, LOGN>(p, a, s)));
  else if (passes & 2)
    KFBI_TRY(kfbi_launch(p, KFBI_K_COLS, s, [&] { cols_real<LOGN><<<4 * a.npl, CT, smem, s>>>(a); }));
  if (passes & 4)
    KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
      rows_inv_real<LOGN><<<a.rows, CT, smem, s>>>(a, static_cast<double *>(u));
    }));
  return KFBI_OK;
}

// FACR(1) for real data at M = 16384 on the one-real-row engine (box_real.cuh).
template <int LOGN>
kfbi_status box_facr_real_launch(kfbi_plan *p, const BoxArgs &a0, const void *rhs, double sign,
                                 const CorrArgs<double> &c, void *u, cudaStream_t s) {
  constexpr int LOGL = LOGN - 1, M = 1 << LOGN;
  static bool attr = false;
  const int bytes = (int)reg::smem_bytes<LOGL>();
  constexpr size_t osm = odd1_smem_bytes<LOGN>();
  if (!attr) {
    KFBI_CUDA(cudaFuncSetAttribute(rows_fwd_facr_real<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
              "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(rows_inv_real<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
              "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(rows_odd_facr_real1<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)osm), "diagonal-scale");
    attr = true;
  }
  CorrArgs<double> cc = c;
  if (c.jv && a0.gsum) {
    double *gs = static_cast<double *>(a0.gsum);
    KFBI_TRY(kfbi_launch(p, KFBI_K_JUMPS, s, [&] { group_sums_kernel<double><<<148 * 2, 256, 0, s>>>(c, M, gs); }));
    cc.cval = gs;
  }
  BoxArgs a = a0;
  a.rows = M / 2;
  a.npl = M / 4;
  a.ring_end = 0;
  a.rowz = a0.zbuf;                                 // zero even rows: flagged, no panels written
  constexpr int CT = reg::Cfg<LOGL>::CTA_T;
  KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
    rows_fwd_facr_real<LOGN><<<M / 2, CT, bytes, s>>>(a, static_cast<const double *>(rhs), sign, cc);
  }));
  BoxArgs ar = a;
  ar.red = 1;
  KFBI_TRY((cols_tri_launch<false, LOGN - 1>(p, ar, s)));
  BoxArgs ai = a;
  ai.row_step = 2;
  KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
    rows_inv_real<LOGN><<<M / 2, CT, bytes, s>>>(ai, static_cast<double *>(u));
  }));
  BoxArgs ao = a0;
  ao.trow = 1;
  ao.tb_re = 1.0 + 0.5 * a0.kre * a0.h2;
  ao.tb_im = 0.0;
  ao.tscale = 1.0;
  if (a0.oc_list) {                                  // trace-only first sweep: the stencil chunks
    if (a0.n_oc == 0) return KFBI_OK;
    return kfbi_launch(p, KFBI_K_SCALE, s, [&] {
      rows_odd_facr_sparse<false, LOGN><<<(a0.n_oc + OS_WARPS - 1) / OS_WARPS, OS_WARPS * 32, 0, s>>>(
          ao, rhs, sign, cc, u);
    });
  }
  return kfbi_launch(p, KFBI_K_SCALE, s, [&] {
    rows_odd_facr_real1<LOGN><<<M / 2, M / 16, osm, s>>>(ao, static_cast<const double *>(rhs), sign, cc,
                                                         static_cast<double *>(u));
  });
}

template <bool CPLX>
kfbi_status box_facr_switch(kfbi_plan *p, int logm, const BoxArgs &a, const void *rhs, double sign,
                            const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                            void *u, cudaStream_t s) {
  switch (logm) {
#define KFBI_CASE(L) \
    case L: return box_facr_launch<CPLX, L>(p, a, rhs, sign, c, u, s);
    KFBI_CASE(6) KFBI_CASE(7) KFBI_CASE(8) KFBI_CASE(9) KFBI_CASE(10) KFBI_CASE(11) KFBI_CASE(12) KFBI_CASE(13)
#undef KFBI_CASE
    case 14:
      if constexpr (!CPLX) return box_facr_real_launch<14>(p, a, rhs, sign, c, u, s);
      return kfbi_fail(KFBI_E_CONFIG, "FACR box solve: complex data at M = 16384 not supported");
    default: return kfbi_fail(KFBI_E_CONFIG, "FACR box solve: 64 <= M <= 8192 (16384 real)");
  }
}

template <bool CPLX>
kfbi_status box_passes_reg(kfbi_plan *p, int logm, bool tri, const BoxArgs &a, const void *rhs, double sign,
                           const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                           void *u, cudaStream_t s, int passes = 7) {
  if (passes == 8) return box_facr_switch<CPLX>(p, logm, a, rhs, sign, c, u, s);   // FACR(1)
  if constexpr (!CPLX) {
    if (logm == 14) return box_real_launch<14>(p, tri, a, rhs, sign, c, u, passes, s);
  }
  switch (logm) {
#define KFBI_CASE(L) \
    case L: return box_reg_launch<CPLX, L>(p, tri, a, rhs, sign, c, u, passes, s);
    KFBI_CASE(4) KFBI_CASE(5) KFBI_CASE(6) KFBI_CASE(7) KFBI_CASE(8) KFBI_CASE(9)
    KFBI_CASE(10) KFBI_CASE(11) KFBI_CASE(12) KFBI_CASE(13) KFBI_CASE(14)
#undef KFBI_CASE
    default: return kfbi_fail(KFBI_E_CONFIG, "register DST engine: unsupported M");
  }
}


// neumann-zero closure: DCT-I passes (box_neu.cuh), one GPU
template <bool CPLX, int LOGN>
kfbi_status box_neu_launch(kfbi_plan *p, const BoxArgs &a, const void *rhs, double sign,
                           const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                           void *u, cudaStream_t s) {
  using Cf = reg::Cfg<LOGN>;
  static bool attr = false;
  if (!attr) {
    const int bytes = (int)reg::smem_bytes<LOGN>();
    KFBI_CUDA(cudaFuncSetAttribute(rows_fwd_neu<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(rows_inv_neu<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-rows");
    KFBI_CUDA(cudaFuncSetAttribute(cols_neu<CPLX, LOGN>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "transform-cols");
    attr = true;
  }
  const int M = Cf::N;
  const int nrow = CPLX ? M + 1 : M / 2 + 1;
  const int ncol = 2 * (CPLX ? M / 2 + 1 : M / 4 + 1);
  const int grow = Cf::CL > 1 ? nrow * Cf::CL : (nrow + Cf::S - 1) / Cf::S;
  const int gcol = Cf::CL > 1 ? ncol * Cf::CL : (ncol + Cf::S - 1) / Cf::S;
  using CT = typename std::conditional<CPLX, double2, double>::type;
  KFBI_TRY(kfbi_launch(p, KFBI_K_ROWS, s, [&] {
    return reg_launch<LOGN>(rows_fwd_neu<CPLX, LOGN>, grow, s, a, rhs, sign, CorrArgs<CT>(c));
  }));
  KFBI_TRY(kfbi_launch(p, KFBI_K_COLS, s, [&] { return reg_launch<LOGN>(cols_neu<CPLX, LOGN>, gcol, s, a); }));
  return kfbi_launch(p, KFBI_K_ROWS, s, [&] { return reg_launch<LOGN>(rows_inv_neu<CPLX, LOGN>, grow, s, a, u); });
}

template <bool CPLX>
kfbi_status box_neu_switch(kfbi_plan *p, int logm, const BoxArgs &a, const void *rhs, double sign,
                           const CorrArgs<typename std::conditional<CPLX, double2, double>::type> &c,
                           void *u, cudaStream_t s) {
  switch (logm) {
#define KFBI_CASE(L) \
    case L: return box_neu_launch<CPLX, L>(p, a, rhs, sign, c, u, s);
    KFBI_CASE(4) KFBI_CASE(5) KFBI_CASE(6) KFBI_CASE(7) KFBI_CASE(8) KFBI_CASE(9)
    KFBI_CASE(10) KFBI_CASE(11) KFBI_CASE(12) KFBI_CASE(13) KFBI_CASE(14)
#undef KFBI_CASE
    default: return kfbi_fail(KFBI_E_CONFIG, "DCT-I engine: unsupported M");
  }
}

}  // namespace kfbi
