// Blackwell (sm_100a) tensor-core plumbing for the certified CROWN contraction:
// tcgen05 MMA (kind::i8, int32 accumulators in TMEM), TMEM allocation and
// loads, TMA tensor-tiled loads (cp.async.bulk.tensor) and the shared-memory
// matrix descriptors of the 128-byte-swizzled K-major operand layout.
//
// Operand tile layout (both A and B): a [rows][128 bytes of K] tile, 1024-byte
// aligned, 16-byte chunk c of row r stored at chunk (c ^ (r & 7)) -- the
// SWIZZLE_128B pattern TMA writes for a {128 B, rows} box and the UMMA
// descriptor (layout type 2, SBO = 1024 B per 8 rows) reads.  One MMA consumes
// K = 32 int8 values; the k-th 32-byte step of a tile is addressed by adding
// 32 k bytes to the descriptor's start address (inside the swizzle atom).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dt_common.cuh"

namespace rb {
namespace tc {

// ---- instruction descriptor (kind::i8): D s32, A/B signed int8, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)                                  // c_format = S32
         | (1u << 7) | (1u << 10)                   // a_format = b_format = signed int8
         | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

// ---- shared-memory matrix descriptor, SWIZZLE_128B K-major (SBO = 1024 B)
__device__ __forceinline__ uint64_t sdesc_sw128(const void* smem_tile) {
  const uint32_t a = smem_u32(smem_tile);
  uint64_t d = 0;
  d |= static_cast<uint64_t>((a >> 4) & 0x3FFFu);          // start address
  d |= static_cast<uint64_t>(1u) << 16;                     // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;             // SBO: 8 rows x 128 B
  d |= static_cast<uint64_t>(1u) << 46;                     // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;                     // SWIZZLE_128B
  return d;
}
// advance a descriptor by `bytes` along K inside the 128-byte atom
__device__ __forceinline__ uint64_t sdesc_add(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }

// byte offset of element (row, k) (k < 128) inside a swizzled K-major tile
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t row, uint32_t k) {
  return row * 128u + ((((k >> 4) ^ (row & 7u)) & 7u) << 4) + (k & 15u);
}

// ---- TMEM allocation (one warp), relinquish, free
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (UMMA operand reads)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- MMA: D[tmem] (+)= A[smem] . B[smem]^T, issued by one thread
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// The same MMA issued by a converged warp: one lane is elected inside the instruction sequence, so
// the warp stays convergent (no per-MMA divergent-branch handling of the uniform operands).
__device__ __forceinline__ void mma_i8_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 r;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` when every previously issued MMA of this thread has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// commit from a converged warp (one elected lane)
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      ".reg .b32 r;\n"
      "elect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// ---- TMEM -> registers: 32 lanes x 16 consecutive 32-bit columns (warp w reads lanes 32 (w % 4) ..)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- TMA: 3-D tensor-tiled load completing on an mbarrier (UTMALDG)
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

}  // namespace tc

// ---------------------------------------------------------------------------
// Ozaki-style exact int8 splitting (the fp64-grade contraction on the int8
// tensor cores).  A row x with scale exponent E (|x_k| < 2^(E-1)) is
//   x_k = 2^E (sum_{t<7} s_t,k 2^-7(t+1) + r_k 2^-49),  |r_k| <= 1/2,  |s_t,k| <= 64,
// with slices s_t from round-to-nearest steps (exact in fp64).  A product of two
// split rows keeps the slice pairs with t + u <= 8 (39 int8 MMAs per 32-wide K
// step, grouped by level g = t + u into 9 exact int32 accumulators); the value is
//   2^(EA + EB - 70) sum_g acc_g 2^(7 (8 - g)),
// and the residuals (2^-50 relative to the row scales) and the dropped pairs
// (levels >= 9: 4 pairs of at most 2^(EA+EB-65) per k, and smaller) are bounded
// per output element by
//   2^-50 (2^EA |b|_1 + 2^EB |a|_1) + K 2^(EA + EB - 62)             (bound).
namespace oz {

constexpr int kSlices = 7;
constexpr int kGroups = 9;  // levels g = t + u = 0 .. 8
constexpr int kPairs = 39;

// scale exponent of a row with max |x| = amax: 2^(E-1) > amax (E = 0 for a zero row)
__host__ __device__ __forceinline__ int scale_exp(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  frexp(amax, &e);  // amax = m 2^e, m in [0.5, 1)  ->  amax < 2^e
  return e + 1;
}

// the 7 slices of x at scale exponent E
__device__ __forceinline__ void split7(double x, int E, int8_t (&s)[kSlices]) {
  double y = ldexp(x, -E);
#pragma unroll
  for (int t = 0; t < kSlices; ++t) {
    y *= 128.0;
    const double q = rint(y);
    y -= q;
    s[t] = static_cast<int8_t>(static_cast<int>(q));
  }
}

// combine the 9 level accumulators of one output element (exact up to the final rounding):
// sum_g acc_g 2^(7 (8 - g)) = hi 2^35 + lo with |hi| < 2^42, |lo| < 2^51
__device__ __forceinline__ double combine(const int32_t (&acc)[kGroups], int ea_eb) {
  const long long hi = ((static_cast<long long>(acc[0]) * 128 + acc[1]) * 128 + acc[2]) * 128 + acc[3];
  const long long lo =
      (((static_cast<long long>(acc[4]) * 128 + acc[5]) * 128 + acc[6]) * 128 + acc[7]) * 128 + acc[8];
  const double v = fma(static_cast<double>(hi), 34359738368.0, static_cast<double>(lo));  // hi 2^35 + lo
  return ldexp(v, ea_eb - 70);
}

// rigorous bound of |a.b - combine(..)| for rows a (scale EA, |a|_1 = l1a) and b over K terms
__host__ __device__ __forceinline__ double bound(int ea, double l1a, int eb, double l1b, int K) {
  if (!(l1a > 0.0) || !(l1b > 0.0)) return 0.0;  // a zero row splits exactly into zero slices
  return ldexp(1.0, -50) * (ldexp(l1b, ea) + ldexp(l1a, eb)) + static_cast<double>(K) * ldexp(1.0, ea + eb - 62);
}

}  // namespace oz
}  // namespace rb
