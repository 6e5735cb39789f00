// Ozaki int8 operand preparation and a standalone certified contraction kernel
// (the building block of the tensor-core CROWN mode, tc_kernel.cuh).
//
//   oz_split_rows_kernel  fp64 rows (M x K, row-major) -> 7 int8 slice planes
//                         [7][Mp][Kp] (zero padded), per-row scale exponent and
//                         |row|_1 -- the layout a TMA tensor map streams as the
//                         A operand (weights are split once, at network upload).
//   oz_gemm_kernel        D = A . B^T (+ the per-element rigorous error bound) for one
//                         128-row M tile per CTA: B rows split in the CTA into
//                         swizzled shared-memory tiles, A tiles streamed by TMA
//                         through a 2-stage mbarrier ring, 39 tcgen05.mma.kind::i8 per
//                         32-wide K step into 9 TMEM accumulators, tcgen05.ld epilogue.
#pragma once

#include "tc_common.cuh"

namespace rb {
namespace oz {

constexpr int kTileRows = 128;   // UMMA M
constexpr int kTileK = 128;      // bytes of K per swizzled tile (one swizzle atom)
constexpr int kTileBytes = kTileRows * kTileK;

__global__ void oz_split_rows_kernel(const double* __restrict__ X, int rows, int K, long long ldx, int Mp, int Kp,
                                     int8_t* __restrict__ planes, int* __restrict__ ex, double* __restrict__ l1) {
  // one warp per row: max / L1 by warp reduction, then the slices
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= Mp) return;
  const int r = warp;
  double amax = 0.0, s1 = 0.0;
  if (r < rows)
    for (int k = lane; k < K; k += 32) {
      const double v = fabs(X[static_cast<long long>(r) * ldx + k]);
      amax = fmax(amax, v);
      s1 += v;
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  const int E = scale_exp(amax);
  if (lane == 0) {
    ex[r] = E;
    l1[r] = s1 * (1.0 + 1e-15);  // rounded up: the L1 norm only enters error bounds
  }
  const size_t plane = static_cast<size_t>(Mp) * Kp;
  for (int k = lane; k < Kp; k += 32) {
    int8_t s[kSlices];
    const double v = (r < rows && k < K) ? X[static_cast<long long>(r) * ldx + k] : 0.0;
    split7(v, E, s);
#pragma unroll
    for (int t = 0; t < kSlices; ++t) planes[t * plane + static_cast<size_t>(r) * Kp + k] = s[t];
  }
}

struct GemmArgs {
  const double* B;  // N x K row-major (fp64)
  int M, N, K, Kp;  // N multiple of 8, <= 56; Kp multiple of 128, <= 256
  const int* ea;    // [Mp] A row scale exponents
  const double* l1a;
  double* D;        // M x N
  double* bnd;      // M x N error bounds
};

// smem: B slices [7][Kp/128][N x 128 B] | A ring [2][16 KB] | barriers | B scales
__global__ void __launch_bounds__(128, 1) oz_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = g.N, nkc = g.Kp / kTileK;
  const int btile = N * kTileK;  // bytes of one (slice, k-chunk) B tile
  unsigned char* bsl = sm;
  unsigned char* aring = sm + ((kSlices * nkc * btile + 1023) & ~1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(aring + 2 * kTileBytes);  // full[2], empty[2], done
  double* l1b = reinterpret_cast<double*>(bar + 8);
  int* eb = reinterpret_cast<int*>(l1b + 64);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eb + 64);
  const int m0 = blockIdx.x * kTileRows;

  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(bar + i, 1);
    fence_mbar_init();
    tc::tma_prefetch(&tmap_a);
  }
  // ---- split the B rows into swizzled K-major tiles
  if (tid < N) {
    double amax = 0.0, s1 = 0.0;
    for (int k = 0; k < g.K; ++k) {
      const double v = fabs(g.B[static_cast<long long>(tid) * g.K + k]);
      amax = fmax(amax, v);
      s1 += v;
    }
    eb[tid] = scale_exp(amax);
    l1b[tid] = s1 * (1.0 + 1e-15);
  }
  __syncthreads();
  for (int e = tid; e < N * g.Kp; e += blockDim.x) {
    const int n = e / g.Kp, k = e - n * g.Kp;
    int8_t s[kSlices];
    split7(k < g.K ? g.B[static_cast<long long>(n) * g.K + k] : 0.0, eb[n], s);
    const uint32_t off = tc::sw128_off(n, k & (kTileK - 1));
#pragma unroll
    for (int t = 0; t < kSlices; ++t) bsl[(t * nkc + (k >> 7)) * btile + off] = static_cast<unsigned char>(s[t]);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (tid == 0) {
    const uint32_t idesc = tc::idesc_i8(kTileRows, N);
    const int total = nkc * kSlices;
    auto issue = [&](int i) {
      const int kc = i / kSlices, t = i - kc * kSlices, s = i & 1;
      mbar_arrive_expect_tx(bar + s, kTileBytes);
      tc::tma_load_3d(aring + s * kTileBytes, &tmap_a, kc * kTileK, m0, t, bar + s);
    };
    for (int i = 0; i < 2 && i < total; ++i) issue(i);
    for (int i = 0; i < total; ++i) {
      const int kc = i / kSlices, t = i - kc * kSlices, s = i & 1;
      mbar_wait(bar + s, (i >> 1) & 1);
      tc::fence_after();
      const uint64_t adesc = tc::sdesc_sw128(aring + s * kTileBytes);
#pragma unroll 1
      for (int kk = 0; kk < kTileK / 32; ++kk) {
        for (int u = 0; u < kSlices && u + t < kGroups; ++u) {
          const uint64_t bdesc = tc::sdesc_sw128(bsl + (u * nkc + kc) * btile);
          tc::mma_i8(tmem + (t + u) * N, tc::sdesc_add(adesc, 32 * kk), tc::sdesc_add(bdesc, 32 * kk), idesc,
                     !(kc == 0 && kk == 0 && (t == 0 || u == kSlices - 1)));  // first write of level t + u
        }
      }
      tc::mma_commit(bar + 2 + s);
      if (i + 2 < total) {
        mbar_wait(bar + 2 + s, (i >> 1) & 1);
        issue(i + 2);
      }
    }
    tc::mma_commit(bar + 4);
  }
  __syncwarp();
  mbar_wait(bar + 4, 0);
  tc::fence_after();
  // ---- epilogue: lane = row m, columns n in groups of 8
  const int m = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  for (int n0 = 0; n0 < N; n0 += 8) {
    int32_t a[kGroups][8];
#pragma unroll
    for (int q = 0; q < kGroups; ++q) tc::tmem_ld8(trow + q * N + n0, a[q]);
    tc::tmem_wait_ld();
    if (m < g.M) {
      const int ea = g.ea[m];
      const double l1 = g.l1a[m];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int n = n0 + j;
        if (n >= N) break;
        int32_t acc[kGroups];
#pragma unroll
        for (int q = 0; q < kGroups; ++q) acc[q] = a[q][j];
        g.D[static_cast<long long>(m) * N + n] = combine(acc, ea + eb[n]);
        g.bnd[static_cast<long long>(m) * N + n] = bound(ea, l1, eb[n], l1b[n], g.K);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 512);
}

// Issue-rate probe: `count` back-to-back MMAs (M = 128, N, K = 32, A and B from shared memory, one
// accumulator; `naccum` > 1 rotates the destination over that many accumulators), timed by thread 0.
__global__ void __launch_bounds__(128, 1) oz_mma_rate_kernel(int count, int N, int naccum, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<int*>(sm)[i] = 0x01010101 * (i & 3);
  if (tid < 32) tc::tmem_alloc(slot, 512);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *slot;
  const int mode = naccum >> 8;
  naccum &= 255;
  if (mode == 0 && tid == 0) {
    const uint32_t idesc = tc::idesc_i8(128, N);
    const uint64_t a = tc::sdesc_sw128(sm), b = tc::sdesc_sw128(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i)
      tc::mma_i8(tmem + (i % naccum) * N, tc::sdesc_add(a, 32 * (i & 3)), tc::sdesc_add(b, 32 * (i & 3)), idesc, 1);
    tc::mma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    cycles[0] = t1 - t0;
  } else if (mode == 1 && tid < 32) {  // converged warp, elected lane inside the asm
    const uint32_t idesc = tc::idesc_i8(128, N);
    const uint64_t a = tc::sdesc_sw128(sm), b = tc::sdesc_sw128(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i)
      tc::mma_i8_warp(tmem + (i % naccum) * N, tc::sdesc_add(a, 32 * (i & 3)), tc::sdesc_add(b, 32 * (i & 3)), idesc,
                      1);
    tc::mma_commit_warp(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (tid == 0) cycles[0] = t1 - t0;
  } else if (mode == 2 && tid == 0) {  // one thread, loop-invariant operands
    const uint32_t idesc = tc::idesc_i8(128, N);
    const uint64_t a = tc::sdesc_sw128(sm), b = tc::sdesc_sw128(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i) tc::mma_i8(tmem, a, b, idesc, 1);
    tc::mma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    cycles[0] = t1 - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) tc::tmem_free(tmem, 512);
}

}  // namespace oz
}  // namespace rb
