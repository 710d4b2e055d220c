// Host-side pieces shared by the translation units of libkfbi_b200.so: error
// reporting, per-launch accounting (the Backend.timings contract of
// engine.py:84-95, kept by the plan in kfbi_b200.cu) and the box-solve entry
// points compiled in their own units (box_dir_*.cu, box_neu_*.cu) so the
// heavy kernel instantiations build in parallel.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <type_traits>

#include "../../include/kfbi_b200.h"
#include "box_kernels.cuh"

kfbi_status kfbi_fail(kfbi_status code, const std::string &msg);

struct KfbiLaunchTok {
  cudaEvent_t a = nullptr, b = nullptr;
};
KfbiLaunchTok kfbi_launch_begin(kfbi_plan *p, int name, cudaStream_t s);
kfbi_status kfbi_launch_end(kfbi_plan *p, int name, cudaStream_t s, KfbiLaunchTok t, cudaError_t e);

// Launch helper: per-name accounting, optional event bracketing and an NVTX
// range named after the kernel family (engine.py:23-35 names).
template <typename F>
kfbi_status kfbi_launch(kfbi_plan *p, int name, cudaStream_t s, F &&fn) {
  KfbiLaunchTok t = kfbi_launch_begin(p, name, s);
  cudaError_t e = cudaSuccess;
  if constexpr (std::is_same<decltype(fn()), cudaError_t>::value) e = fn();
  else fn();
  return kfbi_launch_end(p, name, s, t, e);
}

#define KFBI_CUDA(call, kname)                                                     \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return kfbi_fail(KFBI_E_CUDA, std::string("kernel '") + (kname) + "': " +    \
                                        cudaGetErrorString(_e) + " (" #call ")");  \
  } while (0)

#define KFBI_TRY(expr)                 \
  do {                                 \
    kfbi_status _s = (expr);           \
    if (_s != KFBI_OK) return _s;      \
  } while (0)

// Box-solve passes (boxsolve.py:46-94) for one dtype; `passes` selects any of
// rows_fwd (1), cols (2), rows_inv (4); tri: the tridiagonal column stage.
kfbi_status box_dirichlet_f64(kfbi_plan *p, int logm, bool tri, const kfbi::BoxArgs &a,
                              const void *rhs, double sign, const kfbi::CorrArgs<double> &c,
                              void *u, cudaStream_t s, int passes);
kfbi_status box_dirichlet_c128(kfbi_plan *p, int logm, bool tri, const kfbi::BoxArgs &a,
                               const void *rhs, double sign, const kfbi::CorrArgs<double2> &c,
                               void *u, cudaStream_t s, int passes);
// Transpose-free slab column stage (box_tri.cuh cols_tri_dist); logr = log2
// of the slab rows, units = column units of the dtype.
kfbi_status box_cols_dist(kfbi_plan *p, bool cplx, int logr, const kfbi::BoxArgs &a,
                          const kfbi_tri_dist *d, cudaStream_t s);
kfbi_status box_neumann_f64(kfbi_plan *p, int logm, const kfbi::BoxArgs &a, const void *rhs,
                            double sign, const kfbi::CorrArgs<double> &c, void *u, cudaStream_t s);
kfbi_status box_neumann_c128(kfbi_plan *p, int logm, const kfbi::BoxArgs &a, const void *rhs,
                             double sign, const kfbi::CorrArgs<double2> &c, void *u, cudaStream_t s);
