// Instantiations of the wide kernel family for one rows-per-thread value of
// the dynamics (WIDE_RD, set by the Makefile); compiled as separate objects so
// the family builds in parallel.
#include "wide_kernel.cuh"

#ifndef WIDE_RD
#error "WIDE_RD must be defined"
#endif
#define RB_CAT2(a, b) a##b
#define RB_CAT(a, b) RB_CAT2(a, b)

namespace rb {

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

// P == nullptr: configure the kernel and report CTAs per SM in *occ; else launch.
cudaError_t RB_CAT(wide_call_rd, WIDE_RD)(int rc, const DTParams* P, size_t smem, int grid, int* occ, cudaStream_t s) {
  switch (rc) {
    case 0: return wide_call_t<WIDE_RD, 0>(P, smem, grid, occ, s);
    case 1: return wide_call_t<WIDE_RD, 1>(P, smem, grid, occ, s);
    case 3: return wide_call_t<WIDE_RD, 3>(P, smem, grid, occ, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rb
