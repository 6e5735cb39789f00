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
#include "tcw_kernel.cuh"

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

// Split planes of W_l^T for every contraction layer l = 0 .. L-2 (A operand rows = dims[l], K = dims[l+1]).
static int ensure_oz(reach_ctx* ctx, const reach_net* net) {
  if (net->oz_mem) return REACH_OK;
  const int L = net->L;
  if (L < 2) return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core mode needs a hidden layer");
  rb::OzNet oz{};
  size_t n_e = 0, n_planes = 0;
  for (int l = 0; l + 1 < L; ++l) {
    const int M = net->dims[l], K = net->dims[l + 1];
    if (M > 256 || K > 256) return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core mode: layer widths <= 256");
    oz.mp[l] = (M + 127) / 128 * 128;
    oz.kp[l] = (K + 127) / 128 * 128;
    oz.e_off[l] = static_cast<long long>(n_e);
    n_e += oz.mp[l];
    n_planes += static_cast<size_t>(rb::oz::kSlices) * oz.mp[l] * oz.kp[l];
  }
  const size_t o_map = 0, o_ea = align_up(sizeof(CUtensorMap) * rb::kMaxLayers, 256),
               o_l1 = align_up(o_ea + n_e * sizeof(int), 256), o_pl = align_up(o_l1 + n_e * sizeof(double), 1024),
               bytes = o_pl + n_planes;
  char* mem = nullptr;
  RB_CUDA(cudaMalloc(&mem, bytes));
  oz.tmap = reinterpret_cast<const CUtensorMap*>(mem + o_map);
  oz.ea = reinterpret_cast<const int*>(mem + o_ea);
  oz.l1a = reinterpret_cast<const double*>(mem + o_l1);
  std::vector<CUtensorMap> maps(rb::kMaxLayers);
  std::memset(maps.data(), 0, sizeof(CUtensorMap) * maps.size());
  size_t po = 0;
  for (int l = 0; l + 1 < L; ++l) {
    int8_t* planes = reinterpret_cast<int8_t*>(mem + o_pl + po);
    po += static_cast<size_t>(rb::oz::kSlices) * oz.mp[l] * oz.kp[l];
    const double* X = net->dev.blob + net->dev.wt_off[l];
    rb::oz::oz_split_rows_kernel<<<(oz.mp[l] * 32 + 255) / 256, 256, 0, ctx->stream>>>(
        X, net->dims[l], net->dims[l + 1], net->dev.ldt[l], oz.mp[l], oz.kp[l], planes,
        const_cast<int*>(oz.ea) + oz.e_off[l], const_cast<double*>(oz.l1a) + oz.e_off[l]);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cudaFree(mem);
      return cuda_fail(ctx, e, "oz_split_rows_kernel");
    }
    const int rc = make_slice_tmap(ctx, &maps[l], planes, oz.mp[l], oz.kp[l], rb::oz::kSlices);
    if (rc) {
      cudaFree(mem);
      return rc;
    }
  }
  cudaError_t e = cudaMemcpyAsync(mem + o_map, maps.data(), sizeof(CUtensorMap) * maps.size(),
                                  cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(mem);
    return cuda_fail(ctx, e, "tensor-core planes");
  }
  net->oz_mem = mem;
  net->oz = oz;
  return REACH_OK;
}

void free_oz(reach_net* net) {
  if (net && net->oz_mem) {
    cudaFree(net->oz_mem);
    net->oz_mem = nullptr;
  }
}

int plan_tcw(reach_ctx* ctx, const reach_net* net, const reach_net* ctl, int n, long long B, rb::DTParams& P,
             size_t& smem, int& grid, rb::TcwParams& X) {
  const int l = ctl ? ctl->dims[ctl->L] : 0;
  if (n > rb::tcw::kBRows || l > rb::tcw::kBRows)
    return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core mode: state / control dims <= 72");
  if (P.w_hw > 256) return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core mode: layer widths <= 256");
  int rc = ensure_oz(ctx, net);
  if (rc) return rc;
  X = rb::TcwParams{};
  X.net = net->oz;
  if (ctl) {
    rc = ensure_oz(ctx, ctl);
    if (rc) return rc;
    X.ctl = ctl->oz;
  }
  const int n_i = n + l, nomax = std::max(n, l);
  const int lmax = std::max(net->L, ctl ? ctl->L : 0);
  size_t off = rb::tcw::kU0;
  X.o_relax = static_cast<int>(off);
  off += static_cast<size_t>(std::max(lmax - 1, 1)) * P.w_hw * 4 * 8;
  X.o_misc = static_cast<int>(off);
  const size_t misc = static_cast<size_t>(n + n_i + 2 * n + 3 * nomax + std::max(l, 1) + n + 32) +
                      5 * rb::tcw::kBRows + 2 * rb::kMaxLayers;
  off += misc * 8;
  X.o_int = static_cast<int>(off);
  off += (48 + 2 * rb::tcw::kBRows) * 4 + static_cast<size_t>(std::max(lmax - 1, 1)) * 256;
  off = align_up(off, 64);
  X.o_bar = static_cast<int>(off);
  off += (2 * rb::tcw::kRing + 1) * 8 + 8;
  smem = align_up(off, 128) + 1024;  // + slack for the 1024-byte alignment of the dynamic base
  if (smem > static_cast<size_t>(ctx->max_smem))
    return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core wide kernel working set exceeds shared memory");
  // the lambda rows of a third (first-layer Lambda) and the epilogue partials live in the A ring
  if ((static_cast<size_t>(rb::kWideThreads / 32) * rb::tcw::kNT * rb::tcw::kQ +
       static_cast<size_t>(rb::tcw::kNT) * ((n_i + 1) | 1)) * 8 > static_cast<size_t>(rb::tcw::kARing))
    return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core mode: first layer too wide");
  RB_CUDA(cudaFuncSetAttribute(rb::dt_tcw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  int occ = 0;
  RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rb::dt_tcw_kernel, rb::kWideThreads, smem));
  if (occ < 1) return fail(ctx, REACH_E_UNSUPPORTED, "tensor-core wide kernel does not fit on an SM");
  grid = static_cast<int>(std::min<long long>(B, static_cast<long long>(occ) * ctx->num_sms));
  const size_t need = static_cast<size_t>(grid) * P.wws_stride * 8;
  if (need > ctx->wws_bytes) {
    if (ctx->wws) {
      cudaStreamSynchronize(ctx->stream);
      cudaFree(ctx->wws);
      ctx->wws = nullptr;
      ctx->wws_bytes = 0;
    }
    RB_CUDA(cudaMalloc(&ctx->wws, need));
    ctx->wws_bytes = need;
  }
  P.wws = static_cast<double*>(ctx->wws);
  return REACH_OK;
}

cudaError_t tcw_launch(const rb::DTParams& P, const rb::TcwParams& X, size_t smem, int grid, cudaStream_t s) {
  rb::dt_tcw_kernel<<<grid, rb::kWideThreads, smem, s>>>(P, X);
  return cudaGetLastError();
}

}  // namespace rbh

extern "C" {

int reach_debug_mma_rate(reach_ctx* ctx, int32_t count, int32_t N, int32_t naccum, double* cycles_per_mma) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !cycles_per_mma || count <= 0 || N < 8 || N > 256 || (naccum & 255) < 1 || (naccum & 255) * N > 512)
    return REACH_E_INVALID_ARGUMENT;
  long long* d = nullptr;
  RB_CUDA(cudaMalloc(&d, sizeof(long long)));
  const size_t smem = 65536 + 1024 + 64;
  RB_CUDA(cudaFuncSetAttribute(rb::oz::oz_mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  rb::oz::oz_mma_rate_kernel<<<1, 128, smem, ctx->stream>>>(count, N, naccum, d);
  RB_CUDA(cudaGetLastError());
  long long c = 0;
  RB_CUDA(cudaMemcpyAsync(&c, d, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
  RB_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d);
  *cycles_per_mma = static_cast<double>(c) / count;
  return REACH_OK;
}

int reach_debug_ozaki_gemm(reach_ctx* ctx, int32_t M, int32_t N, int32_t K, const double* A, const double* B,
                           double* D, double* bound) {
  rbh::DeviceGuard device_guard_(ctx);
  if (!ctx || !A || !B || !D || !bound) return REACH_E_INVALID_ARGUMENT;
  // UMMA N at M = 128 (measured on B200, tools/tc_shape_probe.py): 8, 16, 24 and multiples of 16 issue;
  // 40 and 56 raise an illegal instruction.  9 level accumulators x N <= 512 TMEM columns.
  if (M <= 0 || N <= 0 || N > 48 || (N & 7) || (N > 24 && (N & 15)) || K <= 0 || K > 256)
    return fail(ctx, REACH_E_INVALID_ARGUMENT, "ozaki_gemm: need N in {8, 16, 24, 32, 48}, K <= 256");
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
