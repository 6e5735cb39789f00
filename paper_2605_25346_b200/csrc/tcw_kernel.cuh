// Tensor-core precision mode of the wide DT reachability kernel (REACH_PREC_TC):
// certify_tm_input (neural.hpp:342-394) with the dense CROWN contractions
// Lambda <- Lambda_s . W_l (neural.hpp:326) on the 5th-generation tensor cores.
//
// One 256-thread CTA per sample (persistent), as dt_wide_kernel; what changes
// is the backward pass:
//   * Lambda_s rows are split into 7 int8 slices (Ozaki, tc_common.cuh) and
//     written straight into 128-byte-swizzled K-major shared-memory tiles -- the
//     B operand;
//   * the weights W_l^T were split once at network upload; TMA streams their
//     [128 rows x 128 B] slice tiles through a 3-stage mbarrier ring -- the A operand;
//   * one thread issues 39 tcgen05.mma.kind::i8 per 32-wide K step into 9 exact
//     int32 accumulators per output element in TMEM (M = 128 units per tile,
//     N = 24 Lambda rows per pass: a third of the 72-D dynamics' rows, all 18
//     controller rows);
//   * the epilogue (tcgen05.ld) combines the 9 levels into fp64, applies the
//     next layer's relaxation (neural.hpp:166-227) and reduces the intercept and
//     shift chains over the units with warp shuffles -- the chains are fused;
//     the rigorous contraction-error bound (sum_j eps_ij |z_j|_max, z the layer's
//     IBP input box) widens the intercepts, so the result stays a sound
//     over-approximation; then the scaled rows are split into the next B operand.
// IBP, the prepended [A | I] layer (DFMA), re-seed, fold_overflow and symbolic_box
// run on the CUDA cores as in the exact kernel.  Results match the reference to
// ~1e-9 relative (tests/test_gpu_tcw.py), not bit for bit.
#pragma once

#include "tc_common.cuh"
#include "tcw_types.cuh"
#include "wide_kernel.cuh"

namespace rb {

namespace tcw {

constexpr int kNT = 24;                           // Lambda rows per MMA pass (UMMA N)
constexpr int kBRows = 72;                        // max output rows of a net (per-row state arrays)
constexpr int kBTile = kNT * oz::kTileK;          // 3072 B: one (slice, K-chunk) B tile of one third's rows
constexpr int kBBytes = oz::kSlices * 2 * kBTile;  // 7 slices x 2 K-chunks (K <= 256)
constexpr int kRing = 8;
constexpr int kARing = kRing * oz::kTileBytes;
constexpr int kU0 = kBBytes + kARing;             // union region (also IBP / prepend-IBP / fold scratch)
constexpr int kTmemCols = 512;
constexpr int kMTCols = oz::kGroups * kNT;        // TMEM columns per M tile (216)
constexpr int kQ = 5;                             // reduced quantities: lo, up, shift, l1, max

// Pipeline state owned by thread 0 (ring stage counter) and by all threads (done phase).
struct Pipe {
  unsigned char* aring;
  uint64_t* full;   // [kRing]
  uint64_t* empty;  // [kRing]
  uint64_t* done;
  uint32_t tmem;
  unsigned gstage;  // warp 0 only
  unsigned ndone;   // all threads
};

// MMA pass: D[units of layer l's input][24 rows of one third] = W_l^T . Lambda_s^T, all M tiles of
// W_l^T, K = dims[l+1].  Thread 0 issues; every thread returns after the accumulators are complete.
__device__ __forceinline__ void mma_pass(Pipe& pp, const OzNet& oz, int l, int K, const unsigned char* bsl) {
  // Warp 0 issues, converged: one lane is elected inside each MMA / commit (a divergent single-thread
  // issue loop costs ~110 cycles per tcgen05.mma against ~55-64 here, tools/mma_rate.py).
  if (threadIdx.x < 32) {
    const bool lead = threadIdx.x == 0;
    tc::fence_after();
    const CUtensorMap* map = oz.tmap + l;
    const int nmt = oz.mp[l] / oz::kTileRows, nkc = oz.kp[l] / oz::kTileK;
    const int total = nmt * nkc * oz::kSlices;
    const uint32_t idesc = tc::idesc_i8(oz::kTileRows, kNT);
    const unsigned g0 = pp.gstage;
    auto issue = [&](int i) {
      const unsigned g = g0 + i;
      const int s = g % kRing;
      if (lead) {
        if (g >= kRing) mbar_wait(pp.empty + s, ((g - kRing) / kRing) & 1);
        const int t = i % oz::kSlices, kc = (i / oz::kSlices) % nkc, mt = i / (oz::kSlices * nkc);
        mbar_arrive_expect_tx(pp.full + s, oz::kTileBytes);
        tc::tma_load_3d(pp.aring + s * oz::kTileBytes, map, kc * oz::kTileK, mt * oz::kTileRows, t, pp.full + s);
      }
      __syncwarp();
    };
    for (int i = 0; i < kRing - 1 && i < total; ++i) issue(i);
    for (int i = 0; i < total; ++i) {
      const unsigned g = g0 + i;
      const int s = g % kRing;
      if (i + kRing - 1 < total) issue(i + kRing - 1);
      mbar_wait(pp.full + s, (g / kRing) & 1);
      tc::fence_after();
      const int t = i % oz::kSlices, kc = (i / oz::kSlices) % nkc, mt = i / (oz::kSlices * nkc);
      const int ksteps = min(oz::kTileK, K - kc * oz::kTileK + 31) / 32;
      const uint64_t adesc = tc::sdesc_sw128(pp.aring + s * oz::kTileBytes);
      const uint32_t dcol = pp.tmem + mt * kMTCols;
      for (int kk = 0; kk < ksteps; ++kk) {
#pragma unroll
        for (int u = 0; u < oz::kSlices; ++u) {
          if (u + t >= oz::kGroups) break;
          const uint64_t bdesc = tc::sdesc_sw128(bsl + (u * 2 + kc) * kBTile);
          tc::mma_i8_warp(dcol + (t + u) * kNT, tc::sdesc_add(adesc, 32 * kk), tc::sdesc_add(bdesc, 32 * kk), idesc,
                          !(kc == 0 && kk == 0 && (t == 0 || u == oz::kSlices - 1)));  // first write of level t + u
        }
      }
      tc::mma_commit_warp(pp.empty + s);
    }
    tc::mma_commit_warp(pp.done);
    pp.gstage = g0 + total;
  }
  mbar_wait(pp.done, pp.ndone & 1);
  ++pp.ndone;
  tc::fence_after();
}

// Reduce-scatter of 8 columns x kQ quantities over the 32 lanes of a warp: afterwards lane L holds the
// warp totals of column col8(L) = 4 b4 + 2 b3 + b2 (bits of L); quantity kQ-1 is a max, the others sums.
__device__ __forceinline__ int col8(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }
__device__ __forceinline__ void warp_reduce8(double (&v)[kQ][8], int lane, double (&out)[kQ]) {
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    double k4[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double send = b4 ? v[q][c] : v[q][c + 4];
      const double keep = b4 ? v[q][c + 4] : v[q][c];
      const double o = __shfl_xor_sync(0xffffffffu, send, 16);
      k4[c] = (q == kQ - 1) ? fmax(keep, o) : keep + o;
    }
    double k2[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double send = b3 ? k4[c] : k4[c + 2];
      const double keep = b3 ? k4[c + 2] : k4[c];
      const double o = __shfl_xor_sync(0xffffffffu, send, 8);
      k2[c] = (q == kQ - 1) ? fmax(keep, o) : keep + o;
    }
    double k1;
    {
      const double send = b2 ? k2[0] : k2[1];
      const double keep = b2 ? k2[1] : k2[0];
      const double o = __shfl_xor_sync(0xffffffffu, send, 4);
      k1 = (q == kQ - 1) ? fmax(keep, o) : keep + o;
    }
#pragma unroll
    for (int off = 2; off; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, k1, off);
      k1 = (q == kQ - 1) ? fmax(k1, o) : k1 + o;
    }
    out[q] = k1;
  }
}

// Shared-memory views of the TC wide kernel.
struct TSmem {
  unsigned char* bsl;  // B slices [7][2][24 x 128 B] of the current third
  double* red;         // [8 warps][24 rows][kQ] epilogue partials (in the A ring while no MMA runs)
  double* lam0;        // [24][lam0_ld] first-layer Lambda rows of a third (A ring, after red)
  int lam0_ld;
  double* blo;         // [72] per-row intercepts / inflation / scales of the current net
  double* bup;
  double* infl;
  double* l1c;         // [72] |Lambda_s row|_1 of the current B operand
  double* l1n;         // next
  int* ebc;            // [72] scale exponents of the current B rows
  int* ebn;            // next
  double* z1;          // [kMaxLayers] sum_j 2^EA_j zmax_j of GEMM layer l (inputs of W_l)
  double* z2;          // sum_j |W_l^T row j|_1 zmax_j
};

// Relaxation + chains + split of one third of Lambda's rows (r0 .. r0 + nr), given per-thread values
// lam(c) for the unit j of this thread (M tile mt = warp / 4, lane quadrant = warp % 4).
// Phase A reduces the chain contributions over the units; phase B splits Lambda_s into the B operand.
// `getlam(c8, vals[8])` loads 8 consecutive rows' values (chunk c8 of 3) for this thread's unit.
template <class GetLam>
__device__ __forceinline__ bool relax_split_third(const DevNet& N, const WideSmem& W, const TSmem& T, int lrel,
                                                  int width, int r0, int nr, int n_o, bool gemm_out, int Kgemm,
                                                  double z1, double z2, GetLam&& getlam) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = (warp >> 2) * 128 + (warp & 3) * 32 + lane;  // this thread's unit
  const bool uvalid = j < width;
  const int act = N.acts[lrel];
  double s = 0.0, li = 0.0, ui = 0.0, bj = 0.0;
  if (uvalid) {
    const double* R = W.relax + (lrel * W.hw + j) * 4;
    s = R[0];
    li = R[1];
    ui = R[2];
    bj = R[3];
  }
  bool bad = false;
  // ---- phase A: intercept / shift / L1 / max contributions, reduced over the 256 units
  for (int c8 = 0; c8 < 3; ++c8) {
    double lam[8];
    getlam(c8, lam);
    double v[kQ][8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int row = c8 * 8 + c;
      const double a = (uvalid && row < nr) ? lam[c] : 0.0;
      bad |= !finite(a);
      const bool pos = a >= 0.0;
      v[0][c] = a * (pos ? li : ui);
      v[1][c] = a * (pos ? ui : li);
      const double as = (act == 2) ? a : a * s;
      v[2][c] = as * bj;
      v[3][c] = fabs(as);
      v[4][c] = fabs(as);
    }
    double o[kQ];
    warp_reduce8(v, lane, o);
    if ((lane & 3) == 0) {
      const int row = c8 * 8 + col8(lane);
#pragma unroll
      for (int q = 0; q < kQ; ++q) T.red[(warp * kNT + row) * kQ + q] = o[q];
    }
  }
  bad = __syncthreads_or(bad) != 0;
  if (tid < nr) {
    const int i = r0 + tid;
    double lo = 0.0, up = 0.0, sh = 0.0, l1 = 0.0, mx = 0.0;
    for (int w = 0; w < kWideThreads / 32; ++w) {  // fixed order: deterministic
      const double* p = T.red + (w * kNT + tid) * kQ;
      lo += p[0];
      up += p[1];
      sh += p[2];
      l1 += p[3];
      mx = fmax(mx, p[4]);
    }
    T.blo[i] = T.blo[i] + lo + sh;
    T.bup[i] = T.bup[i] + up + sh;
    if (gemm_out)  // sum_j eps_ij zmax_j of the contraction that produced these rows (oz::bound summed over j)
      T.infl[i] += ldexp(1.0, -50) * (T.l1c[i] * z1 + ldexp(z2, T.ebc[i])) +
                   static_cast<double>(Kgemm) * ldexp(z1, T.ebc[i] - 62);
    T.ebn[i] = oz::scale_exp(mx);
    T.l1n[i] = l1 * (1.0 + 1e-15);
    if (!finite(mx) || !finite(l1) || !finite(T.blo[i]) || !finite(T.bup[i])) bad = true;
  }
  if (__syncthreads_or(bad)) return false;
  // ---- phase B: split Lambda_s rows into the next B operand (K index = unit j)
  const int kc = j >> 7, kin = j & 127;
  for (int c8 = 0; c8 < 3; ++c8) {
    double lam[8];
    getlam(c8, lam);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int row = c8 * 8 + c;
      if (row >= kNT) break;
      const bool live = uvalid && row < nr;
      const double a = live ? lam[c] : 0.0;
      const double as = (act == 2) ? a : a * s;
      int8_t sl[oz::kSlices];
      oz::split7(as, live ? T.ebn[r0 + row] : 0, sl);
      const uint32_t off = tc::sw128_off(row, kin);
#pragma unroll
      for (int t = 0; t < oz::kSlices; ++t) T.bsl[(t * 2 + kc) * kBTile + off] = static_cast<unsigned char>(sl[t]);
    }
  }
  tc::fence_async_smem();
  tc::fence_before();  // this thread's tcgen05.ld complete before the next MMA pass reuses TMEM
  __syncthreads();
  return true;
}

// Decoded accumulator values for this thread's TMEM lane: 8 rows (chunk c8) of M tile (warp / 4).
__device__ __forceinline__ void tmem_rows8(uint32_t tmem, int c8, const int* ebc, int r0, int ea, double (&lam)[8]) {
  const int warp = threadIdx.x >> 5;
  const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * kMTCols + c8 * 8;
  int32_t a[oz::kGroups][8];
#pragma unroll
  for (int g = 0; g < oz::kGroups; ++g) tc::tmem_ld8(base + g * kNT, a[g]);
  tc::tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    int32_t acc[oz::kGroups];
#pragma unroll
    for (int g = 0; g < oz::kGroups; ++g) acc[g] = a[g][c];
    lam[c] = oz::combine(acc, ea + ebc[r0 + c8 * 8 + c]);
  }
}

// Block-wide sum of two doubles (result to every thread).
__device__ __forceinline__ void block_sum2(double& a, double& b, double* scratch) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  if (lane == 0) {
    scratch[2 * warp] = a;
    scratch[2 * warp + 1] = b;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
  for (int w = 0; w < kWideThreads / 32; ++w) {
    a += scratch[2 * w];
    b += scratch[2 * w + 1];
  }
  __syncthreads();
}

// certify_tm_input (neural.hpp:342-394) of one sample, tensor-core backward pass.
// Arguments as wide_certify (wide_kernel.cuh).
__device__ int tcw_certify(const DevNet& N, const OzNet& oz, int n_i, int n_o, int nx, const double* u,
                           const double* A, long long lda, int nz, const double* frad, const double* cin, double* out,
                           long long ldo, const WideSmem& W, const TSmem& T, Pipe& pp, WPhase& ph, int pb) {
  const int tid = threadIdx.x;
  const int L = N.L;
  ph.mark(pb + WP_PRE_IBP);
  double2* hin = reinterpret_cast<double2*>(W.lt);
  double2* hout = hin + W.hw;

  // ---- prepend layer IBP (neural.hpp:360-373): the same row abs-sum chains as the exact kernel
  {
    double* sbuf = deep_ring(W.lt, W.hw);
    const long long room = static_cast<long long>(kU0 / 8) - (sbuf - W.lt);
    double hi = 0.0;
    if (room >= 2ll * n_i * 65) {
      hi = row_abs_sums_staged<64>(A, lda, n_i, nz, sbuf);
    } else if (tid < n_i) {
      const double* row = A + tid * lda;
      for (int j = 0; j < nz; ++j) hi = add(hi, fabs(row[j]));
    }
    if (tid < n_i) {
      if (frad && tid >= nx) hi = add(hi, fabs(frad[tid - nx]));
      const double lo = (hi == 0.0) ? 0.0 : -hi;
      const double c = cin[tid];
      hin[tid] = make_double2(add(lo, c), add(hi, c));
    }
    __syncthreads();
    // inflation sums of the first-layer contraction (inputs z = x in hin)
    double a = 0.0, b = 0.0;
    if (tid < n_i) {
      const double zm = fmax(fabs(hin[tid].x), fabs(hin[tid].y));
      a = ldexp(zm, oz.ea[oz.e_off[0] + tid]);
      b = oz.l1a[oz.e_off[0] + tid] * zm;
    }
    block_sum2(a, b, W.red);
    if (tid == 0) {
      T.z1[0] = a * (1.0 + 1e-12);
      T.z2[0] = b * (1.0 + 1e-12);
    }
  }

  // ---- IBP through the hidden layers + relaxation (neural.hpp:166-257), as the exact kernel
  ph.mark(pb + WP_HID_IBP);
  bool bad = false;
  for (int l = 0; l + 1 < L; ++l) {
    const int width = N.dims[l + 1];
    const int act = N.acts[l];
    const unsigned char* inlist = (l == 0) ? nullptr : W.lists + (l - 1) * 256;
    const int nk = (l == 0) ? N.dims[0] : W.cnt[l - 1];
    const int o = tid;
    double alo = 0.0, ahi = 0.0;
    double bfold = (o < width) ? N.blob[N.b_off[l] + o] : 0.0;
    auto ibp_row = [&](const double* row, int j) {
      if (o < width) {
        const double w = row[o];
        if (l == 0 && j >= n_i) {
          bfold = add(bfold, mul(w, u[j - n_i]));
        } else {
          const double2 x = hin[j];
          const bool pos = w >= 0.0;
          alo = add(alo, mul(w, pos ? x.x : x.y));
          ahi = add(ahi, mul(w, pos ? x.y : x.x));
        }
      }
    };
    stream_rows<kDeepNS, kDeepRS>(deep_ring(W.lt, W.hw), N.blob + N.wt_off[l], N.ldt[l], inlist, nk, width, ibp_row);
    bool flag = false;
    double za = 0.0, zb = 0.0;
    if (o < width) {
      const double plo = add(alo, bfold), phi = add(ahi, bfold);
      const bool fin = finite(plo) && finite(phi);
      if (act != 2 && !fin) bad = true;
      double s = 1.0, li = 0.0, ui = 0.0;
      if (act != 2) relax(act, plo, phi, s, li, ui);
      double* R = W.relax + (l * W.hw + o) * 4;
      R[0] = s;
      R[1] = li;
      R[2] = ui;
      R[3] = bfold;
      flag = (act != 0) || plo >= 0.0 || !(phi <= 0.0);
      const double zlo = act_apply(act, plo), zhi = act_apply(act, phi);
      hout[o] = make_double2(zlo, zhi);
      if (l + 2 < L) {  // layer l+1 is a contraction: inflation sums over its inputs z = act(p)
        const double zm = fmax(fabs(zlo), fabs(zhi));
        za = ldexp(zm, oz.ea[oz.e_off[l + 1] + o]);
        zb = oz.l1a[oz.e_off[l + 1] + o] * zm;
      }
    }
    block_compact(flag, o, W.lists + l * 256, W.cnt + l, W.iv + 8);
    if (l + 2 < L) {
      block_sum2(za, zb, W.red);
      if (tid == 0) {
        T.z1[l + 1] = za * (1.0 + 1e-12);
        T.z2[l + 1] = zb * (1.0 + 1e-12);
      }
    }
    double2* t = hin;
    hin = hout;
    hout = t;
  }
  if (__syncthreads_or(bad)) return WC_PREACT;

  // ---- CROWN backward on the tensor cores.  Init: Lambda = W_{L-1}, b = b_{L-1} (neural.hpp:297-305)
  ph.mark(pb + WP_CHAINS);
  const double* Wout = N.blob + N.w_off[L - 1];
  const long long ldo_w = N.ldw[L - 1];
  if (tid < n_o) {
    const double bi = N.blob[N.b_off[L - 1] + tid];
    T.blo[tid] = bi;
    T.bup[tid] = bi;
    T.infl[tid] = 0.0;
  }
  __syncthreads();
  // Depth-first over thirds of Lambda's rows: each third runs the whole backward pass (its B operand
  // holds only its own 24 rows), so the TMA ring can be deep.
  const int nthird = (n_o + kNT - 1) / kNT;
  const int warp = tid >> 5, lane = tid & 31;
  const int j = (warp >> 2) * 128 + (warp & 3) * 32 + lane;  // this thread's unit / TMEM lane
  for (int h = 0; h < nthird; ++h) {
    const int r0 = h * kNT, nr = min(kNT, n_o - r0);
    ph.mark(pb + WP_CHAINS);
    {
      const int lrel = L - 2, width = N.dims[L - 1];
      auto getw = [&](int c8, double (&lam)[8]) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int row = c8 * 8 + c;
          lam[c] = (j < width && row < nr) ? Wout[(r0 + row) * ldo_w + j] : 0.0;
        }
      };
      if (!relax_split_third(N, W, T, lrel, width, r0, nr, n_o, false, 0, 0.0, 0.0, getw)) return WC_CERT;
      if (tid < nr) {  // the B operand now holds Lambda_s of the last hidden layer
        T.ebc[r0 + tid] = T.ebn[r0 + tid];
        T.l1c[r0 + tid] = T.l1n[r0 + tid];
      }
      __syncthreads();
    }
    for (int l = L - 2; l >= 0; --l) {
      const int K = N.dims[l + 1];
      const int width = N.dims[l];  // output units of this contraction (inputs of layer l)
      ph.mark(pb + WP_GEMM);
      mma_pass(pp, oz, l, K, T.bsl);
      ph.mark(pb + (l >= 1 ? WP_CHAINS : WP_PRE_GEMM));
      const int ea = (j < oz.mp[l]) ? oz.ea[oz.e_off[l] + j] : 0;
      const bool tile_live = (warp >> 2) * 128 < oz.mp[l];
      if (l >= 1) {
        auto gett = [&](int c8, double (&lam)[8]) {
          if (tile_live) tmem_rows8(pp.tmem, c8, T.ebc, r0, ea, lam);
          else
            for (int c = 0; c < 8; ++c) lam[c] = 0.0;
        };
        if (!relax_split_third(N, W, T, l - 1, width, r0, nr, n_o, true, K, T.z1[l], T.z2[l], gett)) return WC_CERT;
        if (tid < nr) {
          T.ebc[r0 + tid] = T.ebn[r0 + tid];
          T.l1c[r0 + tid] = T.l1n[r0 + tid];
        }
        __syncthreads();
      } else {
        // ---- first layer: Lambda_0 rows of this third -> lam0; prepended [A | I] layer for these rows
        if (tile_live) {
          for (int c8 = 0; c8 < 3; ++c8) {
            double lam[8];
            tmem_rows8(pp.tmem, c8, T.ebc, r0, ea, lam);
            if (j < n_i)
#pragma unroll
              for (int c = 0; c < 8; ++c) T.lam0[(c8 * 8 + c) * T.lam0_ld + j] = lam[c];
          }
        }
        tc::fence_before();
        __syncthreads();
        bool nf = false;
        if (tid < nr) {
          const int i = r0 + tid;
          T.infl[i] += ldexp(1.0, -50) * (T.l1c[i] * T.z1[0] + ldexp(T.z2[0], T.ebc[i])) +
                       static_cast<double>(K) * ldexp(T.z1[0], T.ebc[i] - 62);
          // shift chain of the prepended layer (b = c): Lambda_0 . cin
          double shv = 0.0;
          for (int k = 0; k < n_i; ++k) {
            const double lv = T.lam0[tid * T.lam0_ld + k];
            nf |= !finite(lv);
            shv = fma(lv, cin[k], shv);
          }
          T.blo[i] += shv;
          T.bup[i] += shv;
        }
        if (__syncthreads_or(nf)) return WC_CERT;
        // out[i][g] = sum_k Lambda_0[i][k] A[k][g] (DFMA, rows of this third), generator g per thread;
        // the A column is loaded 8 rows ahead of the FMAs (global-latency bound otherwise)
        for (int g = tid; g < nz; g += kWideThreads) {
          double acc[kNT];
#pragma unroll
          for (int c = 0; c < kNT; ++c) acc[c] = 0.0;
          for (int k0 = 0; k0 < n_i; k0 += 8) {
            double av[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) av[q] = (k0 + q < n_i) ? A[(k0 + q) * lda + g] : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (k0 + q >= n_i) break;
              const double* lr = T.lam0 + k0 + q;
#pragma unroll
              for (int c = 0; c < kNT; ++c) acc[c] = fma(lr[c * T.lam0_ld], av[q], acc[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < kNT; ++c)
            if (c < nr) out[(r0 + c) * ldo + g] = acc[c];
        }
        if (frad)
          for (int e = tid; e < nr * n_i; e += kWideThreads) {
            const int c = e / n_i, jj = e - c * n_i;
            out[(r0 + c) * ldo + nz + jj] = (jj < nx) ? 0.0 : T.lam0[c * T.lam0_ld + jj] * frad[jj - nx];
          }
        __syncthreads();
      }
    }
  }
  // ---- tail (neural.hpp:383-391), intercepts widened by the contraction-error bound
  bool rbad = false;
  if (tid < n_o) {
    const double blo = T.blo[tid] - T.infl[tid], bup = T.bup[tid] + T.infl[tid];
    const double mid = (blo + bup) * 0.5;
    const double rl = blo - mid, rh = bup - mid;
    W.mid[tid] = mid;
    W.rl[tid] = rl;
    W.rh[tid] = rh;
    rbad = !(finite(rl) && finite(rh));
  }
  return __syncthreads_or(rbad) ? WC_CERT : WC_OK;
}

}  // namespace tcw

// The TC wide horizon kernel: dt_wide_kernel (wide_kernel.cuh) with tcw_certify.
__global__ void __launch_bounds__(kWideThreads, 1) dt_tcw_kernel(const DTParams P, const TcwParams X) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  double* sd = reinterpret_cast<double*>(sm);
  const int tid = threadIdx.x;
  const int n = P.n, m = P.m, H = P.H, lc = P.l;
  const int n_i = n + lc;
  const int cap = P.window > 0 ? P.window : 1;
  const int nomax = max(n, lc);
  WideSmem W;
  W.nop = 1;
  W.hw = P.w_hw;
  W.lt = sd;  // U0: IBP buffers / prepend-IBP staging / fold scratch (outside the backward pass)
  W.stages = nullptr;
  W.relax = reinterpret_cast<double*>(sm + X.o_relax);
  W.bf0 = nullptr;
  double* ms = reinterpret_cast<double*>(sm + X.o_misc);
  W.cst = ms;
  W.cag = W.cst + n;
  W.xlo = W.cag + n_i;
  W.xhi = W.xlo + n;
  W.mid = W.xhi + n;
  W.rl = W.mid + nomax;
  W.rh = W.rl + nomax;
  W.urad = W.rh + nomax;
  W.radv = W.urad + (lc > 0 ? lc : 1);
  W.red = W.radv + n;
  tcw::TSmem T;
  T.bsl = sm;
  T.red = reinterpret_cast<double*>(sm + tcw::kBBytes);
  T.lam0 = T.red + (kWideThreads / 32) * tcw::kNT * tcw::kQ;
  T.lam0_ld = ((n_i > 0 ? n_i : 1) + 1) | 1;
  T.blo = W.red + 32;
  T.bup = T.blo + tcw::kBRows;
  T.infl = T.bup + tcw::kBRows;
  T.l1c = T.infl + tcw::kBRows;
  T.l1n = T.l1c + tcw::kBRows;
  T.z1 = T.l1n + tcw::kBRows;
  T.z2 = T.z1 + kMaxLayers;
  int* is = reinterpret_cast<int*>(sm + X.o_int);
  W.wid = is;
  W.iv = is + 16;
  W.cnt = is + 32;
  T.ebc = is + 48;
  T.ebn = T.ebc + tcw::kBRows;
  W.lists = reinterpret_cast<unsigned char*>(T.ebn + tcw::kBRows);
  W.bars = nullptr;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + X.o_bar);
  tcw::Pipe pp;
  pp.aring = sm + tcw::kBBytes;
  pp.full = bars;
  pp.empty = bars + tcw::kRing;
  pp.done = bars + 2 * tcw::kRing;
  pp.gstage = 0;
  pp.ndone = 0;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * tcw::kRing + 1);
  if (tid < 32) tc::tmem_alloc(tmem_slot, tcw::kTmemCols);
  if (tid == 0) {
    for (int i = 0; i < 2 * tcw::kRing + 1; ++i) mbar_init(bars + i, 1);
    fence_mbar_init();
    for (int l = 0; l + 1 < P.net.L; ++l) tc::tma_prefetch(X.net.tmap + l);
    if (lc > 0)
      for (int l = 0; l + 1 < P.ctl.L; ++l) tc::tma_prefetch(X.ctl.tmap + l);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pp.tmem = *tmem_slot;

  const long long lds = P.w_lds;
  double* buf0 = P.wws + static_cast<long long>(blockIdx.x) * P.wws_stride;
  double* buf1 = buf0 + static_cast<long long>(P.w_rows) * lds;
  WPhase ph{P.w_phase, clock64(), WP_SETUP};

  for (long long b = blockIdx.x; b < P.B; b += gridDim.x) {
    const double* act_base = P.actions;
    if (!P.actions_shared && m > 0) act_base += static_cast<size_t>(b) * H * m;
    if (tid < n) {
      double lo, hi;
      if (P.split) {
        split_edges(P, P.part_begin + b, tid, lo, hi);
      } else if (P.x0_center) {
        const double c = P.x0_lo[tid];
        lo = sub(c, P.x0_eps);
        hi = add(c, P.x0_eps);
      } else {
        lo = P.x0_lo[b * n + tid];
        hi = P.x0_hi[b * n + tid];
      }
      W.xlo[tid] = lo;
      W.xhi[tid] = hi;
    }
    __syncthreads();
    auto emit_box = [&](int k, bool all_fin) {
      if (tid >= n) return;
      const double lo = W.xlo[tid], hi = W.xhi[tid];
      if (!P.split) {
        const size_t o = (static_cast<size_t>(b) * (H + 1) + k) * n + tid;
        P.out_lo[o] = lo;
        P.out_hi[o] = hi;
      } else {
        if (lo == lo) atomicMin(&P.hull_lo[k * n + tid], order_key(lo));
        if (hi == hi) atomicMax(&P.hull_hi[k * n + tid], order_key(hi));
        if (P.part_begin + b == 0) {
          if (lo != lo) P.hull_nan0[(k * n + tid) * 2 + 0] = 1;
          if (hi != hi) P.hull_nan0[(k * n + tid) * 2 + 1] = 1;
        }
        if (!all_fin && tid == 0) atomicOr(&P.hull_div[k], 1);
      }
    };
    double* cur = buf0;
    double* oth = buf1;
    int base = 0, nq = 0;
    auto init_state = [&]() {
      for (int e = tid; e < n * n; e += kWideThreads) {
        const int i = e / n, j = e - i * n;
        cur[i * lds + j] = (i == j) ? mul(sub(W.xhi[i], W.xlo[i]), 0.5) : 0.0;
      }
      if (tid < n) W.cst[tid] = mul(add(W.xlo[tid], W.xhi[tid]), 0.5);
      base = 0;
      nq = 0;
      __syncthreads();
    };
    {
      const bool f = (tid >= n) || (finite(W.xlo[tid]) && finite(W.xhi[tid]));
      const bool all_fin = __syncthreads_and(f) != 0;
      emit_box(0, all_fin);
    }
    init_state();
    int status = ST_OK, failed_step = -1, nboxes = 1;

    for (int k = 0; k < H; ++k) {
      int nz = n;
      for (int q = 0; q < nq; ++q) nz += W.wid[q];
      const double* u = act_base + static_cast<size_t>(k) * m;
      const double* cin = W.cst;
      const double* frad = nullptr;
      if (lc > 0) {
        const int rc = tcw::tcw_certify(P.ctl, X.ctl, n, lc, n, nullptr, cur + base, lds, nz, nullptr, W.cst,
                                        cur + n * lds + base, lds, W, T, pp, ph, 0);
        if (rc != WC_OK) {
          status = (rc == WC_PREACT) ? ST_CTL_PREACT : ST_CTL_CERT;
          failed_step = k;
          break;
        }
        if (tid < lc) {
          W.urad[tid] = mul(sub(W.rh[tid], W.rl[tid]), 0.5);
          W.cag[n + tid] = add(W.mid[tid], mul(add(W.rl[tid], W.rh[tid]), 0.5));
        }
        if (tid < n) W.cag[tid] = add(W.cst[tid], 0.0);
        __syncthreads();
        cin = W.cag;
        frad = W.urad;
      }
      const int rc =
          tcw::tcw_certify(P.net, X.net, n_i, n, n, u, cur + base, lds, nz, frad, cin, oth, lds, W, T, pp, ph, 5);
      if (rc != WC_OK) {
        status = (rc == WC_PREACT) ? ST_PREACT : ST_CERT;
        failed_step = k;
        break;
      }
      // ---- re-seed (dt_reach.hpp:69-92)
      ph.mark(WP_RESEED);
      const int nza = nz + (lc > 0 ? n_i : 0);
      if (tid < n) {
        W.cst[tid] = add(W.mid[tid], mul(add(W.rl[tid], W.rh[tid]), 0.5));
        W.radv[tid] = mul(sub(W.rh[tid], W.rl[tid]), 0.5);
      }
      if (tid == 0) {
        if (lc > 0) W.wid[nq] = n_i;
        W.wid[nq + (lc > 0 ? 1 : 0)] = n;
      }
      __syncthreads();
      for (int e = tid; e < n * n; e += kWideThreads) {
        const int i = e / n, j = e - i * n;
        oth[i * lds + nza + j] = (i == j) ? W.radv[i] : 0.0;
      }
      nq += (lc > 0) ? 2 : 1;
      base = 0;
      {
        double* t = cur;
        cur = oth;
        oth = t;
      }
      __syncthreads();
      // ---- fold_overflow (flowpipe_ct.hpp:317-350)
      ph.mark(WP_FOLD);
      wide_fold<72>(cur, lds, n, base, nq, cap, W, ph);
      // ---- symbolic_box (flowpipe_ct.hpp:413-424)
      ph.mark(WP_BOX);
      bool fin = true;
      if (tid < n) {
        const double* row = cur + tid * lds + base;
        double r = 0.0;
        for (int j = 0; j < n; ++j) r = add(r, fabs(row[j]));
        int off = n;
        for (int q = 0; q < nq; ++q) {
          double s = 0.0;
          const int wq = W.wid[q];
          for (int j = 0; j < wq; ++j) s = add(s, fabs(row[off + j]));
          r = add(r, s);
          off += wq;
        }
        const double c = W.cst[tid];
        const double lo = sub(c, r), hi = add(c, r);
        W.xlo[tid] = lo;
        W.xhi[tid] = hi;
        fin = finite(lo) && finite(hi);
      }
      const bool all_fin = __syncthreads_and(fin) != 0;
      emit_box(k + 1, all_fin);
      nboxes = k + 2;
      if (!all_fin) {
        status = ST_BOX;
        failed_step = k;
        break;
      }
      if (P.rebuild) init_state();
      ph.mark(WP_SETUP);
    }
    __syncthreads();
    if (tid == 0) {
      if (!P.split) {
        P.n_boxes[b] = nboxes;
        P.failed_step[b] = failed_step;
        P.status[b] = status;
      } else {
        atomicMin(P.hull_nboxes, nboxes);
        if (status != ST_OK) {
          const unsigned long long key =
              (static_cast<unsigned long long>(failed_step >= 0 ? failed_step : nboxes) << 40) |
              (static_cast<unsigned long long>(P.part_begin + b) << 8) | static_cast<unsigned long long>(status & 0xff);
          atomicMin(P.hull_fail_key, key);
        }
      }
    }
    __syncthreads();
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) tc::tmem_free(pp.tmem, tcw::kTmemCols);
}

}  // namespace rb
