// REACH_PREC_FUSED: the warp-per-sample DT horizon kernel and the wide (CTA-per-sample) family
// compiled a second time with RB_FUSED (dt_common.cuh): every a*b+c of the contractions, IBP
// and chains becomes one DFMA.  Same algorithm, layout and shared-memory carve-up as the exact
// build; the kernels live in namespace rbf (the `rb` token is renamed for this unit only) so the
// two builds link side by side.  The host passes its rb::DTParams, which is layout-identical.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#ifndef WIDE_RD
#error "WIDE_RD must be defined"
#endif

#define RB_FUSED 1
#define rb rbf
#include "wide_kernel.cuh"
#undef rb

#define RB_CAT2(a, b) a##b
#define RB_CAT(a, b) RB_CAT2(a, b)

namespace rbf {

template <int RD, int RC>
static cudaError_t wide_call_t(const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s) {
  auto k = dt_wide_kernel<RD, RC>;
  if (!P) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, kWideThreads, smem);
  }
  k<<<grid, kWideThreads, smem, s>>>(*P);
  return cudaGetLastError();
}

template <int NO, int CPL>
static cudaError_t horizon_t(const DTParams& P, unsigned grid, unsigned threads, size_t smem, cudaStream_t s) {
  auto k = dt_horizon_kernel<NO, CPL>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  k<<<grid, threads, smem, s>>>(P);
  return cudaGetLastError();
}

template <int NO>
static cudaError_t horizon_no(int cpl, const DTParams& P, unsigned grid, unsigned threads, size_t smem,
                              cudaStream_t s) {
  switch (cpl) {
    case 1: return horizon_t<NO, 1>(P, grid, threads, smem, s);
    case 2: return horizon_t<NO, 2>(P, grid, threads, smem, s);
    case 3: return horizon_t<NO, 3>(P, grid, threads, smem, s);
    case 4: return horizon_t<NO, 4>(P, grid, threads, smem, s);
    default: return horizon_t<NO, 8>(P, grid, threads, smem, s);
  }
}

}  // namespace rbf

namespace rbh {

// P: the host's rb::DTParams (same layout as rbf::DTParams); nullptr = configure and report occupancy.
cudaError_t RB_CAT(wide_call_fused_rd, WIDE_RD)(int rc, const void* P, size_t smem, int grid, int* occ,
                                                cudaStream_t s) {
  const rbf::DTParams* p = static_cast<const rbf::DTParams*>(P);
  switch (rc) {
    case 0: return rbf::wide_call_t<WIDE_RD, 0>(p, smem, grid, occ, s);
    case 1: return rbf::wide_call_t<WIDE_RD, 1>(p, smem, grid, occ, s);
    case 3: return rbf::wide_call_t<WIDE_RD, 3>(p, smem, grid, occ, s);
    default: return cudaErrorInvalidValue;
  }
}

#if WIDE_RD == 1
// The warp-per-sample horizon kernel lives in the rd1 unit (one copy).
size_t fused_params_size() { return sizeof(rbf::DTParams); }
cudaError_t launch_dt_fused(const void* P, int no, int cpl, unsigned grid, unsigned threads, size_t smem,
                            cudaStream_t s) {
  const rbf::DTParams& p = *static_cast<const rbf::DTParams*>(P);
  switch (no) {
    case 2: return rbf::horizon_no<2>(cpl, p, grid, threads, smem, s);
    case 4: return rbf::horizon_no<4>(cpl, p, grid, threads, smem, s);
    case 6: return rbf::horizon_no<6>(cpl, p, grid, threads, smem, s);
    default: return rbf::horizon_no<8>(cpl, p, grid, threads, smem, s);
  }
}
#endif

}  // namespace rbh
