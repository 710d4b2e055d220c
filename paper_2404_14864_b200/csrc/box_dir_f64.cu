// Dirichlet-zero box-solve passes, f64 (boxsolve.py:46-94): its own
// translation unit so the kernel instantiations compile in parallel.
#include "box_launch.cuh"

kfbi_status box_dirichlet_f64(kfbi_plan *p, int logm, bool tri, const kfbi::BoxArgs &a,
                              const void *rhs, double sign, const kfbi::CorrArgs<double> &c,
                              void *u, cudaStream_t s, int passes) {
  return kfbi::box_passes_reg<false>(p, logm, tri, a, rhs, sign, c, u, s, passes);
}

// Transpose-free slab column stage (cols_tri_dist), both dtypes.
namespace {
template <bool CPLX, int LOGR>
kfbi_status cols_dist_launch(kfbi_plan *p, const kfbi::BoxArgs &a, const kfbi_tri_dist *dd, cudaStream_t s) {
  using Tc = kfbi::tri::Cfg<LOGR>;
  kfbi::TriDist d;
  d.P = dd->nranks;
  d.g = dd->rank;
  d.virt = dd->virt;
  d.epoch = dd->epoch;
  d.max_spins = dd->max_spins;
  d.timed_out = dd->timed_out;
  const int npl = CPLX ? a.m / 2 : a.m / 4;
  d.units = Tc::NH == 2 ? npl : 2 * npl;
  for (int h = 0; h < 8; ++h) {
    d.vpanels[h] = h < d.P ? dd->panels[h] : nullptr;
    d.agg[h] = h < d.P ? static_cast<double2 *>(dd->agg[h]) : nullptr;
    d.flg[h] = h < d.P ? static_cast<unsigned long long *>(dd->flags[h]) : nullptr;
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  KFBI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfbi::cols_tri_dist<CPLX, LOGR>,
                                                          Tc::THREADS, 0), "transform-cols");
  const int ny = d.virt ? d.P : 1;
  int gx = per_sm * sms / ny;
  if (gx > d.units) gx = d.units;
  if (gx < 1) return kfbi_fail(KFBI_E_CONFIG, "slab column stage: no resident CTAs for the virtual ranks");
  kfbi::BoxArgs aa = a;
  void *args[] = {&aa, &d};
  return kfbi_launch(p, KFBI_K_COLS, s, [&] {
    return cudaLaunchCooperativeKernel((const void *)kfbi::cols_tri_dist<CPLX, LOGR>, dim3(gx, ny),
                                       dim3(Tc::THREADS), args, 0, s);
  });
}
}  // namespace

kfbi_status box_cols_dist(kfbi_plan *p, bool cplx, int logr, const kfbi::BoxArgs &a,
                          const kfbi_tri_dist *d, cudaStream_t s) {
  switch (logr) {
#define KFBI_CASE(L) \
    case L: return cplx ? cols_dist_launch<true, L>(p, a, d, s) : cols_dist_launch<false, L>(p, a, d, s);
    KFBI_CASE(4) KFBI_CASE(5) KFBI_CASE(6) KFBI_CASE(7) KFBI_CASE(8) KFBI_CASE(9)
    KFBI_CASE(10) KFBI_CASE(11) KFBI_CASE(12) KFBI_CASE(13) KFBI_CASE(14)
#undef KFBI_CASE
    default: return kfbi_fail(KFBI_E_CONFIG, "slab column stage: unsupported slab height");
  }
}
