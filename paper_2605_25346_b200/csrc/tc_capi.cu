// Host side of the tensor-core (Ozaki int8) contraction: TMA tensor maps over
// split operand planes, and the debug entry point that runs one certified
// contraction (tests/test_gpu_tc.py checks it against numpy fp64).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <vector>

#include "ctx.cuh"
#include "tc_capi.h"
#include "tc_gemm.cuh"

using namespace rbh;

namespace rbh {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_slice_tmap(reach_ctx* ctx, CUtensorMap* map, const int8_t* planes, int Mp, int Kp, int slices) {
  auto fn = encode_fn();
  if (!fn) return fail(ctx, REACH_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp),
                              static_cast<cuuint64_t>(slices)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(Mp) * Kp};
  const cuuint32_t box[3] = {rb::oz::kTileK, rb::oz::kTileRows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(planes), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, REACH_E_CUDA, "cuTensorMapEncodeTiled failed");
  return REACH_OK;
}

}  // namespace rbh

extern "C" {

int reach_debug_ozaki_gemm(reach_ctx* ctx, int32_t M, int32_t N, int32_t K, const double* A, const double* B,
                           double* D, double* bound) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !A || !B || !D || !bound) return REACH_E_INVALID_ARGUMENT;
  if (M <= 0 || N <= 0 || N > 64 || (N & 7) || K <= 0 || K > 256)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ozaki_gemm: need N in 8..64 (multiple of 8), K <= 256");
  const int Mp = (M + 127) / 128 * 128, Kp = (K + 127) / 128 * 128;
  const size_t planes = static_cast<size_t>(rb::oz::kSlices) * Mp * Kp;
  double *dA, *dB, *dD, *dE, *dl1;
  int8_t* dP;
  int* dex;
  RB_CUDA(cudaMalloc(&dA, sizeof(double) * M * K));
  RB_CUDA(cudaMalloc(&dB, sizeof(double) * N * K));
  RB_CUDA(cudaMalloc(&dD, sizeof(double) * M * N));
  RB_CUDA(cudaMalloc(&dE, sizeof(double) * M * N));
  RB_CUDA(cudaMalloc(&dl1, sizeof(double) * Mp));
  RB_CUDA(cudaMalloc(&dex, sizeof(int) * Mp));
  RB_CUDA(cudaMalloc(&dP, planes));
  RB_CUDA(cudaMemcpyAsync(dA, A, sizeof(double) * M * K, cudaMemcpyHostToDevice, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(dB, B, sizeof(double) * N * K, cudaMemcpyHostToDevice, ctx->stream));
  rb::oz::oz_split_rows_kernel<<<(Mp * 32 + 255) / 256, 256, 0, ctx->stream>>>(dA, M, K, K, Mp, Kp, dP, dex, dl1);
  RB_CUDA(cudaGetLastError());
  CUtensorMap map;
  int rc = make_slice_tmap(ctx, &map, dP, Mp, Kp, rb::oz::kSlices);
  if (rc) return rc;
  rb::oz::GemmArgs g{dB, M, N, K, Kp, dex, dl1, dD, dE};
  const int nkc = Kp / rb::oz::kTileK;
  const size_t smem = 1024 + ((rb::oz::kSlices * nkc * N * rb::oz::kTileK + 1023) & ~size_t(1023)) +
                      2 * rb::oz::kTileBytes + 64 + 64 * 4 + 64 * 8;
  RB_CUDA(cudaFuncSetAttribute(rb::oz::oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  rb::oz::oz_gemm_kernel<<<Mp / 128, 128, smem, ctx->stream>>>(map, g);
  RB_CUDA(cudaGetLastError());
  RB_CUDA(cudaMemcpyAsync(D, dD, sizeof(double) * M * N, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaMemcpyAsync(bound, dE, sizeof(double) * M * N, cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  ++ctx->launches;
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dE);
  cudaFree(dl1);
  cudaFree(dex);
  cudaFree(dP);
  return REACH_OK;
}

}  // extern "C"
