// Wide DT reachability kernel family for B200 (sm_100a): one CTA per sample.
//
// The warp-per-sample horizon kernel (dt_kernel.cuh) keeps a sample's whole
// symbolic state in shared memory, which caps it at n <= 8 and 64 generator
// columns.  The 72-D closed loop (n = 72, l = 18, 3 x 256 ReLU
// dynamics and controller, ~400 generators) needs 150 KB for Lambda alone, so
// here a 256-thread CTA owns one sample at a time (persistent over the batch):
//   * Lambda^T (n_o x width) lives in shared memory; the dense contraction
//     Lambda <- Lambda_s . W_l is a CTA-wide register-tiled product (rows i =
//     warp + 8r, columns j = lane + 32c), its B operand -- the rows k of W_l
//     with a non-zero slope, or the generator rows of the input TM -- streamed
//     through a cp.async ring;
//   * the symbolic state (c, [G0 | Q1 .. Qnq] for x and the controller's u rows)
//     lives in ONE buffer per CTA in global memory (L2-resident): the certified
//     output overwrites its input in place (column j from column base + j);
//     fold_overflow runs as a CTA-parallel partial-pivot elimination in shared
//     memory; popping the oldest block moves G0 right instead of moving the queue.
// Every reduction keeps the reference's order with separate roundings, so the
// results are bit-identical to the warp kernel and to the reference.
#pragma once

#include "dt_common.cuh"
#include "dt_kernel.cuh"

namespace rb {

constexpr int kWideThreads = 256;
#ifndef RB_WIDE_NS
#define RB_WIDE_NS 3
#endif
#ifndef RB_WIDE_RS
#define RB_WIDE_RS 8
#endif
#ifndef RB_WIDE_UNROLL
#define RB_WIDE_UNROLL 4
#endif
constexpr int kWideUnroll = RB_WIDE_UNROLL;  // unroll of the per-row functor over a full stage
constexpr int kWideNS = RB_WIDE_NS;  // cp.async ring stages
constexpr int kWideRS = RB_WIDE_RS;  // rows per stage
constexpr int kWideSW = 256;  // stage row stride (doubles): widest streamed row segment
constexpr int kWideMaxL = kMaxLayers;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Optional phase timing: thread 0 charges the cycles since the last mark to
// the running phase (phases are CTA-synchronous); enabled by a non-null P.w_phase.
struct WPhase {
  unsigned long long* out;
  long long last;
  int cur;
  __device__ __forceinline__ void mark(int next) {
    if (out && threadIdx.x == 0) {
      const long long now = clock64();
      atomicAdd(out + cur, static_cast<unsigned long long>(now - last));
      last = now;
      cur = next;
    }
  }
};
enum : int {
  WP_SETUP = 0, WP_PRE_IBP = 1, WP_HID_IBP = 2, WP_CHAINS = 3, WP_GEMM = 4, WP_PRE_GEMM = 5,  // + 5 for the dynamics
  WP_RESEED = 11, WP_FOLD = 12, WP_BOX = 13, WP_FOLD_ELIM = 14, WP_FOLD_BACK = 15
};

// Shared-memory views of one CTA.
struct WideSmem {
  double* lt;       // Lambda^T [hw][nop]; IBP interval buffers; fold scratch (spans lt..relax)
  double* stages;   // [kWideNS][kWideRS][kWideSW]
  double* relax;    // [L-1][hw][3]  (s, li, ui) per hidden unit
  double* bf0;      // [hw] first-layer bias with the frozen inputs folded in
  double* cst;      // [n]   state centre
  double* cag;      // [n+l] stacked centre
  double* xlo;      // [n]
  double* xhi;      // [n]
  double* mid;      // [max(n,l)] certification tail
  double* rl;
  double* rh;
  double* urad;     // [l]
  double* radv;     // [n]
  double* red;      // [32] reduction scratch
  int* wid;         // [16] generator block widths
  int* iv;          // [16] misc ints (pivot, flags)
  int* cnt;         // [kMaxLayers] active-unit counts
  unsigned char* lists;  // [L-1][256] active units
  uint64_t* bars;        // [8] mbarriers of the bulk-copy rings (null: element-wise cp.async rings)
  int nop, hw;
};

// Streams rows list[0..nk) (identity when list == nullptr) of a row-major
// global matrix -- `ncols` doubles from base + k * ld -- through a cp.async
// ring of NS stages of RS rows and calls f(row_in_smem, k) on every thread, in order.
//
// With `bars` (and 16-byte aligned rows), each row of a chunk is one bulk copy (the TMA engine's 1-D
// form, UBLKCP) completing on the stage's mbarrier: one lane per row issues, instead of every thread
// issuing 8-byte cp.async per element (13 % of the C5 kernel's instructions).
template <int NS = kWideNS, int RS = kWideRS, class F>
__device__ __forceinline__ void stream_rows(double* stages, const double* base, long long ld,
                                            const unsigned char* list, int nk, int ncols, F&& f,
                                            uint64_t* bars = nullptr) {
  const int nch = (nk + RS - 1) / RS;
  static_assert(NS <= 8, "one mbarrier per stage");
  if (bars && nch > 0 &&
      ((reinterpret_cast<uintptr_t>(base) | static_cast<uintptr_t>(ld * 8) | static_cast<uintptr_t>(ncols * 8)) & 15u) ==
          0) {
    const int tid = threadIdx.x;
    __syncthreads();  // the previous user of the barriers and of the stages is done
    if (tid == 0) {
      for (int q = 0; q < NS; ++q) mbar_init(bars + q, 1);
      fence_mbar_init();
    }
    __syncthreads();
    const uint32_t rowb = static_cast<uint32_t>(ncols) * 8u;
    auto bissue = [&](int c) {  // warp 0: lane 0 arms the stage, lanes < nr copy one row each
      if (c < nch && tid < 32) {
        double* st = stages + (c % NS) * (RS * kWideSW);
        const int t0 = c * RS;
        const int nr = min(RS, nk - t0);
        if (tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(bars + c % NS, rowb * static_cast<uint32_t>(nr));
        }
        __syncwarp();
        for (int rr = tid; rr < nr; rr += 32) {
          const int k = list ? static_cast<int>(list[t0 + rr]) : t0 + rr;
          bulk_g2s(st + rr * kWideSW, base + static_cast<long long>(k) * ld, rowb, bars + c % NS);
        }
      }
    };
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) bissue(c);
    for (int c = 0; c < nch; ++c) {
      mbar_wait(bars + c % NS, (c / NS) & 1);
      __syncthreads();  // every thread is past chunk c - 1: its stage can be refilled
      bissue(c + NS - 1);
      const double* st = stages + (c % NS) * (RS * kWideSW);
      const int t0 = c * RS;
      const int nr = min(RS, nk - t0);
      if (nr == RS) {
#pragma unroll kWideUnroll
        for (int rr = 0; rr < RS; ++rr) f(st + rr * kWideSW, list ? static_cast<int>(list[t0 + rr]) : t0 + rr);
      } else {
        for (int rr = 0; rr < nr; ++rr) f(st + rr * kWideSW, list ? static_cast<int>(list[t0 + rr]) : t0 + rr);
      }
    }
    __syncthreads();
    return;
  }
  auto issue = [&](int c) {
    if (c < nch) {
      double* st = stages + (c % NS) * (RS * kWideSW);
      const int t0 = c * RS;
      const int nr = min(RS, nk - t0);
      for (int col = threadIdx.x; col < ncols; col += kWideThreads)
        for (int rr = 0; rr < nr; ++rr) {
          const int k = list ? static_cast<int>(list[t0 + rr]) : t0 + rr;
          cp_async8(st + rr * kWideSW + col, base + static_cast<long long>(k) * ld + col);
        }
    }
    cp_commit();
  };
#pragma unroll
  for (int c = 0; c < NS - 1; ++c) issue(c);
  for (int c = 0; c < nch; ++c) {
    cp_wait<NS - 2>();
    __syncthreads();
    issue(c + NS - 1);
    const double* st = stages + (c % NS) * (RS * kWideSW);
    const int t0 = c * RS;
    const int nr = min(RS, nk - t0);
    if (nr == RS) {
#pragma unroll kWideUnroll
      for (int rr = 0; rr < RS; ++rr) f(st + rr * kWideSW, list ? static_cast<int>(list[t0 + rr]) : t0 + rr);
    } else {
      for (int rr = 0; rr < nr; ++rr) f(st + rr * kWideSW, list ? static_cast<int>(list[t0 + rr]) : t0 + rr);
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// Deep ring for the IBP passes, which have little arithmetic per streamed row:
// while the forward pass runs, Lambda's region is free (after the interval buffers).
constexpr int kDeepNS = 4, kDeepRS = 16;
__device__ __forceinline__ bool deep_ring_fits(int nop, int hw) {
  return static_cast<long long>(nop) * hw >= 4ll * hw + 8 + static_cast<long long>(kDeepNS) * kDeepRS * kWideSW;
}
__device__ __forceinline__ double* deep_ring(double* lt, int hw) { return lt + ((4 * hw + 7) & ~7); }

// Row abs-sums of the input TM, hi_i = sum_j |A_ij| in column order, with the
// rows staged through shared memory in double-buffered column blocks of CB
// (padded row stride CB + 1: conflict-free per-row reads).  The prepend IBP's
// lower chain is its exact negation (round-to-nearest is sign-symmetric).
template <int CB>
__device__ __forceinline__ double row_abs_sums_staged(const double* A, long long lda, int n_i, int nz, double* buf) {
  const int tid = threadIdx.x;
  const int nblk = (nz + CB - 1) / CB;
  const int bstride = n_i * (CB + 1);
  auto issue = [&](int bk) {
    if (bk < nblk) {
      const int c0 = bk * CB, nc = min(CB, nz - c0);
      double* dst = buf + (bk & 1) * bstride;
      for (int e = tid; e < n_i * CB; e += kWideThreads) {
        const int i = e / CB, j = e - i * CB;
        if (j < nc) cp_async8(dst + i * (CB + 1) + j, A + i * lda + c0 + j);
      }
    }
    cp_commit();
  };
  issue(0);
  double hi = 0.0;
  for (int bk = 0; bk < nblk; ++bk) {
    issue(bk + 1);
    cp_wait<1>();
    __syncthreads();
    if (tid < n_i) {
      const double* row = buf + (bk & 1) * bstride + tid * (CB + 1);
      const int nc = min(CB, nz - bk * CB);
#pragma unroll 8
      for (int j = 0; j < nc; ++j) hi = add(hi, fabs(row[j]));
    }
    __syncthreads();
  }
  return hi;
}

// acc[r][c] = sum_k Lambda[warp + 8r][k] * B[k][lane + 32c] over the streamed
// rows k, each a sequential chain in stream order (linalg.hpp:53-63, i-k-j).
template <int RPT, int CPL>
__device__ __forceinline__ void wide_gemm(const double* LT, int nop, double* stages, const double* base, long long ld,
                                          const unsigned char* list, int nk, int ncols, double (&acc)[RPT][CPL],
                                          uint64_t* bars = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[r][c] = 0.0;
  stream_rows(stages, base, ld, list, nk, ncols, [&](const double* row, int k) {
    double lam[RPT], w[CPL];
    const double* lk = LT + k * nop + warp;
#pragma unroll
    for (int r = 0; r < RPT; ++r) lam[r] = lk[8 * r];
#pragma unroll
    for (int c = 0; c < CPL; ++c) w[c] = row[lane + 32 * c];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[r][c] = add(acc[r][c], mul(lam[r], w[c]));
  }, bars);
}

// Lambda <- Lambda_s . W (ncols <= 256) written back into LT; returns true if any
// entry is non-finite (the reference's remainder would be non-finite).
template <int RPT, int CPL>
__device__ __forceinline__ bool gemm_to_lt_t(uint64_t* bars, double* LT, int nop, int n_o, double* stages, const double* W,
                                             long long ldw, const unsigned char* list, int nk, int ncols) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[RPT][CPL];
  wide_gemm<RPT, CPL>(LT, nop, stages, W, ldw, list, nk, ncols, acc, bars);
  bool bad = false;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = warp + 8 * r, j = lane + 32 * c;
      if (i < n_o && j < ncols) {
        LT[j * nop + i] = acc[r][c];
        bad |= !finite(acc[r][c]);
      }
    }
  return __syncthreads_or(bad) != 0;
}

template <int RPT>
__device__ __forceinline__ bool gemm_to_lt(uint64_t* bars, double* LT, int nop, int n_o, double* stages, const double* W, long long ldw,
                                           const unsigned char* list, int nk, int ncols) {
  if (ncols <= 64) return gemm_to_lt_t<RPT, 2>(bars, LT, nop, n_o, stages, W, ldw, list, nk, ncols);
  if (ncols <= 128) return gemm_to_lt_t<RPT, 4>(bars, LT, nop, n_o, stages, W, ldw, list, nk, ncols);
  return gemm_to_lt_t<RPT, 8>(bars, LT, nop, n_o, stages, W, ldw, list, nk, ncols);
}

template <int RPT, int CPL>
__device__ __forceinline__ void gemm_to_global_t(uint64_t* bars, const double* LT, int nop, int n_o, double* stages, const double* A,
                                                 long long lda, int nk, int ncols, double* out, long long ldo) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[RPT][CPL];
  wide_gemm<RPT, CPL>(LT, nop, stages, A, lda, nullptr, nk, ncols, acc, bars);
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int i = warp + 8 * r, j = lane + 32 * c;
      if (i < n_o && j < ncols) out[i * ldo + j] = acc[r][c];
    }
}

// out[:, 0:nz) = Lambda (n_o x nk) . A (nk x nz), in column passes of <= 256.
template <int RPT>
__device__ __forceinline__ void gemm_to_global(uint64_t* bars, const double* LT, int nop, int n_o, double* stages, const double* A,
                                               long long lda, int nk, int nz, double* out, long long ldo) {
  for (int col0 = 0; col0 < nz; col0 += kWideSW) {
    const int nc = min(kWideSW, nz - col0);
    if (nc <= 64) gemm_to_global_t<RPT, 2>(bars, LT, nop, n_o, stages, A + col0, lda, nk, nc, out + col0, ldo);
    else if (nc <= 128) gemm_to_global_t<RPT, 4>(bars, LT, nop, n_o, stages, A + col0, lda, nk, nc, out + col0, ldo);
    else gemm_to_global_t<RPT, 8>(bars, LT, nop, n_o, stages, A + col0, lda, nk, nc, out + col0, ldo);
  }
}

// Order-preserving compaction of the units with flag set (ascending unit index).
__device__ __forceinline__ void block_compact(bool flag, int unit, unsigned char* list, int* count, int* scratch) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) scratch[warp] = __popc(m);
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWideThreads / 32; ++w) {
    const int c = scratch[w];
    if (w < warp) base += c;
    tot += c;
  }
  if (flag) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<unsigned char>(unit);
  if (threadIdx.x == 0) *count = tot;
  __syncthreads();
}

enum : int { WC_OK = 0, WC_PREACT = 1, WC_CERT = 2 };

// certify_tm_input (neural.hpp:342-394) of one sample by the whole CTA.
// Input TM rows 0..n_i-1 of A (row stride lda, nz generator columns; rows
// >= nx additionally own a fresh diagonal generator frad[i - nx] at column
// nz + i when frad != nullptr -- the stacked [x; u] of closed_loop.hpp:118-153),
// centre cin.  N.dims[0] - n_i trailing inputs are frozen to u
// (freeze_trailing_inputs, neural.hpp:398-413).  Writes out[i][0..nz(+n_i))
// = (Lambda . [A | F])_i and the tail (mid, rem) into W.mid / W.rl / W.rh.
template <int RPT>
__device__ int wide_certify(const DevNet& N, int n_i, int n_o, int nx, const double* u, const double* A, long long lda,
                            int nz, const double* frad, const double* cin, double* out, long long ldo,
                            const WideSmem& W, WPhase& ph, int pb) {
  const int tid = threadIdx.x;
  const int L = N.L;
  const int nop = W.nop;
  double* LT = W.lt;
  double2* hin = reinterpret_cast<double2*>(W.lt);
  double2* hout = hin + W.hw;

  // ---- prepend layer IBP (neural.hpp:360-373, interval.hpp:284-295):
  // iv_scale(a, [-1, 1]) = [-|a|, |a|], so the two chains are negations of each other
  ph.mark(pb + WP_PRE_IBP);
  {
    double* sbuf = deep_ring(W.lt, W.hw);
    const long long room = static_cast<long long>(nop) * W.hw - (sbuf - W.lt);
    double hi = 0.0;
    if (room >= 2ll * n_i * 65) {
      hi = row_abs_sums_staged<64>(A, lda, n_i, nz, sbuf);
    } else if (room >= 2ll * n_i * 17) {
      hi = row_abs_sums_staged<16>(A, lda, n_i, nz, sbuf);
    } else if (tid < n_i) {
      const double* row = A + tid * lda;
      for (int j = 0; j < nz; ++j) hi = add(hi, fabs(row[j]));
    }
    if (tid < n_i) {
      if (frad && tid >= nx) hi = add(hi, fabs(frad[tid - nx]));
      const double lo = (hi == 0.0) ? 0.0 : -hi;  // the lower chain of +-0 terms stays +0
      const double c = cin[tid];
      hin[tid] = make_double2(add(lo, c), add(hi, c));
    }
    __syncthreads();
  }

  // ---- IBP through the hidden layers + relaxation (neural.hpp:166-257)
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
    if (deep_ring_fits(nop, W.hw))
      stream_rows<kDeepNS, kDeepRS>(deep_ring(W.lt, W.hw), N.blob + N.wt_off[l], N.ldt[l], inlist, nk, width, ibp_row,
                                    W.bars);
    else
      stream_rows(W.stages, N.blob + N.wt_off[l], N.ldt[l], inlist, nk, width, ibp_row, W.bars);
    bool flag = false;
    if (o < width) {
      const double plo = add(alo, bfold), phi = add(ahi, bfold);
      const bool fin = finite(plo) && finite(phi);
      if (act != 2 && !fin) bad = true;
      double s = 1.0, li = 0.0, ui = 0.0;
      if (act != 2) relax(act, plo, phi, s, li, ui);
      double* R = W.relax + (l * W.hw + o) * 4;  // (s, li, ui, b') per unit
      R[0] = s;
      R[1] = li;
      R[2] = ui;
      R[3] = bfold;
      flag = (act != 0) || plo >= 0.0 || !(phi <= 0.0);
      hout[o] = make_double2(act_apply(act, plo), act_apply(act, phi));
    }
    block_compact(flag, o, W.lists + l * 256, W.cnt + l, W.iv + 8);
    double2* t = hin;
    hin = hout;
    hout = t;
  }
  if (__syncthreads_or(bad)) return WC_PREACT;

  // ---- CROWN backward (neural.hpp:297-327).  Init: Lambda = I . W_{L-1}; b = I . b_{L-1}
  double blo = 0.0, bup = 0.0;
  {
    const int lw = (L == 1) ? n_i : N.dims[L - 1];
    const double* Wl = N.blob + N.w_off[L - 1];
    const long long ld = N.ldw[L - 1];
    for (int e = tid; e < n_o * lw; e += kWideThreads) {
      const int i = e / lw, j = e - i * lw;
      LT[j * nop + i] = add(0.0, Wl[i * ld + j]);
    }
    if (tid < n_o) {
      double bi = N.blob[N.b_off[L - 1] + tid];
      if (L == 1)  // single-layer net: fold the frozen inputs into the bias here
        for (int j = n_i; j < N.dims[0]; ++j) bi = add(bi, mul(Wl[tid * ld + j], u[j - n_i]));
      blo = add(0.0, bi);
      bup = blo;
    }
    __syncthreads();
  }
  for (int l = L - 2; l >= 0; --l) {
    const int act = N.acts[l];
    const unsigned char* list = W.lists + l * 256;
    const int cnt = W.cnt[l];
    const double* R = W.relax + l * W.hw * 4;
    ph.mark(pb + WP_CHAINS);
    if (tid < n_o) {
      // intercept chains, slope scaling and the shift chain of row i, in unit
      // order; operands of 8 units are loaded ahead of their chained updates
      const int i = tid;
      double shift = 0.0;
      constexpr int QB = 8;
      for (int t0 = 0; t0 < cnt; t0 += QB) {
        int jq[QB];
        double aq[QB];
        double4 rq[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          jq[q] = (t0 + q < cnt) ? list[t0 + q] : list[t0];
          aq[q] = LT[jq[q] * nop + i];
          const double2 r01 = *reinterpret_cast<const double2*>(R + 4 * jq[q]);
          const double2 r23 = *reinterpret_cast<const double2*>(R + 4 * jq[q] + 2);
          rq[q] = make_double4(r01.x, r01.y, r23.x, r23.y);
        }
        // branch-free updates: the skipped terms of the reference are +-0 (zero-sign only)
        if (act == 0) {
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            const double a = aq[q];
            const double s = rq[q].x, ui = rq[q].z, bj = rq[q].w;
            const bool live = t0 + q < cnt;
            const double t = mul(a, ui);
            const double nu = add(bup, t), nl = add(blo, t);
            const bool unst = live && ui != 0.0;  // unstable ReLU: li = 0, only the ui side contributes
            bup = (unst && a >= 0.0) ? nu : bup;
            blo = (unst && !(a >= 0.0)) ? nl : blo;
            const double as = mul(a, s);
            if (live) LT[jq[q] * nop + i] = as;
            const double ns = add(shift, mul(as, bj));
            shift = live ? ns : shift;
          }
        } else {
#pragma unroll
          for (int q = 0; q < QB; ++q) {
            if (t0 + q < cnt) {
              const double a = aq[q];
              const double s = rq[q].x, li = rq[q].y, ui = rq[q].z, bj = rq[q].w;
              if (act == 1) {
                const bool pos = a >= 0.0;
                blo = add(blo, mul(a, pos ? li : ui));
                bup = add(bup, mul(a, pos ? ui : li));
              }
              const double as = (act == 2) ? a : mul(a, s);
              LT[jq[q] * nop + i] = as;
              shift = add(shift, mul(as, bj));
            }
          }
        }
      }
      blo = add(blo, shift);
      bup = add(bup, shift);
    }
    __syncthreads();
    ph.mark(pb + WP_GEMM);
    const int ncols = (l == 0) ? n_i : N.dims[l];
    if (gemm_to_lt<RPT>(W.bars, LT, nop, n_o, W.stages, N.blob + N.w_off[l], N.ldw[l], list, cnt, ncols)) return WC_CERT;
  }

  // ---- prepended layer W = [A | I], b = c: shift chain, then Lambda . A
  ph.mark(pb + WP_PRE_GEMM);
  if (tid < n_o) {
    double shift = 0.0;
    for (int k = 0; k < n_i; ++k) shift = add(shift, mul(LT[k * nop + tid], cin[k]));
    blo = add(blo, shift);
    bup = add(bup, shift);
  }
  gemm_to_global<RPT>(W.bars, LT, nop, n_o, W.stages, A, lda, n_i, nz, out, ldo);
  if (frad)
    for (int e = tid; e < n_o * n_i; e += kWideThreads) {
      const int i = e / n_i, jj = e - i * n_i;
      out[i * ldo + nz + jj] = (jj < nx) ? 0.0 : add(0.0, mul(LT[jj * nop + i], frad[jj - nx]));
    }
  // ---- tail (neural.hpp:383-391)
  bool rbad = false;
  if (tid < n_o) {
    const double mid = mul(add(blo, bup), 0.5);
    const double rl = sub(blo, mid), rh = sub(bup, mid);
    W.mid[tid] = mid;
    W.rl[tid] = rl;
    W.rh[tid] = rh;
    rbad = !(finite(rl) && finite(rh));
  }
  return __syncthreads_or(rbad) ? WC_CERT : WC_OK;
}

// Row-wise copy of an n x nc block (global row stride lds) into shared memory
// (row stride nc): every element in flight at once through cp.async.
__device__ __forceinline__ void load_block(double* M, const double* Sb, long long lds, int n, int nc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < n; i += kWideThreads / 32) {
    const double* src = Sb + i * lds;
    double* dst = M + i * nc;
    for (int j = lane; j < nc; j += 32) cp_async8(dst + j, src + j);
  }
  cp_commit();
  cp_wait<0>();
}

// Back substitution of mat_solve (linalg.hpp:125-131) with the solution column in registers: xb[q] = x_{n-1-q};
// row r from the bottom (i = n - 1 - r) subtracts a_{i,k} x_k for k = i + 1 .. n - 1, i.e. q = r - 1 .. 0.
// Fused mode: four partial sums over k >= i + 2 (as the generic fused loop), exact: the reference's chain
// (used by the fused build only, see wide_fold).
// One row of it per template instance (R = rows from the bottom), so every index into xb is a constant
// and the column stays in registers.
template <int R, int NMAX>
struct BackRow {
  static __device__ __forceinline__ void run(double (&xb)[NMAX], const double* M, const int* Pf, double* X, int n,
                                             int nc, int w, int jc) {
    if (R < n) {
      const int i = n - 1 - R;
      const double* mr = M + Pf[i] * nc + (n - 1);  // mr[-q] = a_{i, n-1-q}
      const double bi = mr[1 + jc];
#if RB_FUSED
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int q = R - 2; q >= 0; q -= 4) {
        s0 = fma(mr[-q], xb[q], s0);
        if (q >= 1) s1 = fma(mr[-(q - 1)], xb[q - 1], s1);
        if (q >= 2) s2 = fma(mr[-(q - 2)], xb[q - 2], s2);
        if (q >= 3) s3 = fma(mr[-(q - 3)], xb[q - 3], s3);
      }
      double acc = bi - ((s0 + s1) + (s2 + s3));
      if (R >= 1) acc = fma(-mr[-(R - 1)], xb[R >= 1 ? R - 1 : 0], acc);
      xb[R] = acc / mr[-R];
#else
      double acc = bi;
#pragma unroll
      for (int q = R - 1; q >= 0; --q) acc = sub(acc, mul(mr[-q], xb[q]));
      xb[R] = __ddiv_rn(acc, mr[-R]);
#endif
      X[i * w + jc] = xb[R];
      BackRow<R + 1, NMAX>::run(xb, M, Pf, X, n, nc, w, jc);
    }
  }
};
template <int NMAX>
struct BackRow<NMAX, NMAX> {
  static __device__ __forceinline__ void run(double (&)[NMAX], const double*, const int*, double*, int, int, int, int) {}
};

template <int NMAX>
__device__ __forceinline__ void backsub_regs(const double* M, const int* Pf, double* X, int n, int nc, int w, int tid) {
#if RB_FUSED
  // fused build: rows unrolled by the compiler (the template-recursive form hung in this build; kept as measured)
  for (int jc = tid; jc < w; jc += kWideThreads) {
    double xb[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r) {
      xb[r] = 0.0;
      if (r < n) {
        const int i = n - 1 - r;
        const double* mr = M + Pf[i] * nc + (n - 1);
        const double bi = mr[1 + jc];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int q = r - 2; q >= 0; q -= 4) {
          s0 = fma(mr[-q], xb[q], s0);
          if (q >= 1) s1 = fma(mr[-(q - 1)], xb[q - 1], s1);
          if (q >= 2) s2 = fma(mr[-(q - 2)], xb[q - 2], s2);
          if (q >= 3) s3 = fma(mr[-(q - 3)], xb[q - 3], s3);
        }
        double acc = bi - ((s0 + s1) + (s2 + s3));
        if (r >= 1) acc = fma(-mr[-(r - 1)], xb[r - 1], acc);
        xb[r] = acc / mr[-r];
        X[i * w + jc] = xb[r];
      }
    }
  }
#else
  for (int jc = tid; jc < w; jc += kWideThreads) {
    double xb[NMAX];
    BackRow<0, NMAX>::run(xb, M, Pf, X, n, nc, w, jc);
  }
#endif
}

// fold_overflow (flowpipe_ct.hpp:317-350) on the state in S (rows 0..n-1, row
// stride lds, live columns [base, base + nz)).  Popping the oldest block moves
// the (possibly rescaled) G0 right by its width instead of moving the queue.
template <int NMAX>
static __device__ void wide_fold(double* S, long long lds, int n, int& base, int& nq, int cap, const WideSmem& W,
                                 WPhase& ph) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  while (nq > cap) {
    const int w = W.wid[0];
    const int nc = n + w;
    double* M = W.lt;           // [n][nc]: [G0 | a], eliminated in place; later [G0 | E]
    double* X = M + n * nc;     // [n][w]
    double* rr = X + n * w;     // [n]
    double* F = rr + n;         // [2][n] multipliers of the current / next step
    int* Pm = reinterpret_cast<int*>(F + 2 * n);  // [2][n] logical -> physical row of M
    double* Bst = W.red + 16;   // [2] pivot magnitude of the current / next step
    double* Sb = S + base;
    int off_new = n;
    for (int q = 0; q + 1 < nq; ++q) off_new += W.wid[q];
    load_block(M, Sb, lds, n, nc);
    if (tid < n) Pm[n + tid] = tid;
    __syncthreads();
    ph.mark(WP_FOLD_ELIM);
    // ---- mat_solve (linalg.hpp:96-132): partial pivoting, first maximum wins.
    // Row swaps act on a permutation (the values are those of the reference's
    // swapped rows).  Warp 0 updates the next pivot column, chooses the next
    // pivot and computes its multipliers while the other warps update the rest,
    // so each elimination step costs one barrier.
    // pivot(k): v[t] = column-k values of logical rows k + lane + 32t under perm pin.
    auto pivot = [&](int k, const double (&v)[4], const int* pin, int* pout, double* fout, double* bout) {
      const double vk = __shfl_sync(0xffffffffu, v[0], 0);
      double bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = k + lane + 32 * t;
        if (i > k && i < n) {
          const double a = fabs(v[t]);
          if (a > bv) {
            bv = a;
            bi = i;
          }
        }
      }
      {
        // warp argmax on (|a|, -row) with three redux.sync (342 -> ~100 cycles against five
        // shuffle rounds, tools/ubench/lat_chain.cu): |a| >= 0 orders as its IEEE bits; a lane
        // without a candidate sends key 0 (= +0.0), which never beats |a_kk| either
        const unsigned long long key =
            (bv >= 0.0) ? static_cast<unsigned long long>(__double_as_longlong(bv)) : 0ull;
        const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        bi = __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? bi : 0x7fffffff);
        bv = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(mhi) << 32) | mlo));
      }
      int piv = k;
      double best = fabs(vk);
      if (bv > best) {  // NaN |a_kk|: nothing beats it and the pivot test fails, as the reference
        best = bv;
        piv = bi;
      }
      // value of the pivot row (owner lane (piv - k) % 32, slot (piv - k) / 32)
      const int d = piv - k;
      double vp = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double x = __shfl_sync(0xffffffffu, v[t], d & 31);
        if ((d >> 5) == t) vp = x;
      }
      for (int i = lane; i < n; i += 32) pout[i] = (i == k) ? pin[piv] : (i == piv) ? pin[k] : pin[i];
#if RB_FUSED
      const double rvp = 1.0 / vp;  // fused mode: one reciprocal per pivot
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = k + lane + 32 * t;
        if (i > k && i < n) fout[i] = (i == piv ? vk : v[t]) * rvp;
      }
#else
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = k + lane + 32 * t;
        if (i > k && i < n) fout[i] = __ddiv_rn(i == piv ? vk : v[t], vp);
      }
#endif
      if (lane == 0) *bout = best;
    };
    if (warp == 0) {
      double v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int i = lane + 32 * t;
        v[t] = (i < n) ? M[i * nc] : 0.0;
      }
      pivot(0, v, Pm + n, Pm, F, Bst);
    }
    __syncthreads();
    bool ok = true;
    for (int kk = 0; kk < n; ++kk) {
      const int cb = kk & 1, nb = cb ^ 1;
      if (!(Bst[cb] > 1e-12)) {
        ok = false;
        break;
      }
      if (kk == n - 1) break;
      const int* Pk = Pm + cb * n;
      const double* Fk = F + cb * n;
      const int prow = Pk[kk];
      if (warp == 0) {
        // next pivot column kk+1: a_ij -= f_i a_kj for rows i > kk, then pivot(kk+1)
        const double mk = M[prow * nc + kk + 1];
        double v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int i = kk + 1 + lane + 32 * t;
          v[t] = 0.0;
          if (i < n) {
            double* mp = M + Pk[i] * nc + kk + 1;
            v[t] = sub(*mp, mul(Fk[i], mk));
            *mp = v[t];
          }
        }
        pivot(kk + 1, v, Pk, Pm + nb * n, F + nb * n, Bst + nb);
      } else {
        // columns kk+2 .. nc-1 (the rest of G0 and the right-hand sides), rows > kk in chunks of 8
        const int cols = nc - kk - 2, rows = n - kk - 1;
        const int nchk = (rows + 7) >> 3;
        for (int q = tid - 32; q < cols * nchk; q += kWideThreads - 32) {
          const int ch = q / cols;
          const int j = kk + 2 + (q - ch * cols);
          const double mk = M[prow * nc + j];
          const int i0 = kk + 1 + ch * 8;
          int pr[8];
          double f[8], m[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) pr[r] = (i0 + r < n) ? Pk[i0 + r] : -1;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            f[r] = (pr[r] >= 0) ? Fk[i0 + r] : 0.0;
            m[r] = (pr[r] >= 0) ? M[pr[r] * nc + j] : 0.0;
          }
#pragma unroll
          for (int r = 0; r < 8; ++r)
            if (pr[r] >= 0) M[pr[r] * nc + j] = sub(m[r], mul(f[r], mk));
        }
      }
      __syncthreads();
    }
    const int* Pf = Pm + ((n - 1) & 1) * n;
    bool folded = false;
    ph.mark(WP_FOLD_BACK);
    if (ok) {
      if constexpr (NMAX == 72) {
        // C5-class states (33 <= n <= 72): the solution column held per thread in registers, rows and products
        // unrolled (back substitution per C5 reach-step: fused 173 k -> 105 k cycles, exact 165 k -> 126 k)
        backsub_regs<NMAX>(M, Pf, X, n, nc, w, tid);
      } else
      // back substitution, one RHS column per thread; x_{i+1} stays in a
      // register, the older x_k are read in blocks of 4 ahead of the chain
      for (int jc = tid; jc < w; jc += kWideThreads) {
        double xprev = 0.0;
#if RB_FUSED
        // fused mode: four partial sums per row (a different association; the chain length drops 4x)
        for (int i = n - 1; i >= 0; --i) {
          const double* mrow = M + Pf[i] * nc;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int k = i + 2;
          for (; k + 4 <= n; k += 4) {
            s0 = fma(mrow[k], X[k * w + jc], s0);
            s1 = fma(mrow[k + 1], X[(k + 1) * w + jc], s1);
            s2 = fma(mrow[k + 2], X[(k + 2) * w + jc], s2);
            s3 = fma(mrow[k + 3], X[(k + 3) * w + jc], s3);
          }
          for (; k < n; ++k) s0 = fma(mrow[k], X[k * w + jc], s0);
          double acc = mrow[n + jc] - ((s0 + s1) + (s2 + s3));
          if (i + 1 < n) acc = fma(-mrow[i + 1], xprev, acc);
          xprev = acc / mrow[i];
          X[i * w + jc] = xprev;
        }
        continue;
#endif
        for (int i = n - 1; i >= 0; --i) {
          const double* mrow = M + Pf[i] * nc;
          double acc = mrow[n + jc];
          int k = i + 1;
          if (k < n) {
            acc = sub(acc, mul(mrow[k], xprev));
            ++k;
          }
          for (; k + 4 <= n; k += 4) {
            const double a0 = mrow[k], a1 = mrow[k + 1], a2 = mrow[k + 2], a3 = mrow[k + 3];
            const double x0 = X[k * w + jc], x1 = X[(k + 1) * w + jc], x2 = X[(k + 2) * w + jc],
                         x3 = X[(k + 3) * w + jc];
            acc = sub(acc, mul(a0, x0));
            acc = sub(acc, mul(a1, x1));
            acc = sub(acc, mul(a2, x2));
            acc = sub(acc, mul(a3, x3));
          }
          for (; k < n; ++k) acc = sub(acc, mul(mrow[k], X[k * w + jc]));
          xprev = __ddiv_rn(acc, mrow[i]);
          X[i * w + jc] = xprev;
        }
      }
      __syncthreads();
      double v = 0.0;
      if (tid < n) {
        double s = 0.0;
        for (int c = 0; c < w; ++c) s = add(s, fabs(X[tid * w + c]));
        const double r = mul(s, 1.0 + 1e-12);
        rr[tid] = r;
        v = (r == r) ? r : 0.0;  // std::max(worst, r) never adopts a NaN
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, off));
      if (lane == 0) W.red[1 + warp] = v;
      __syncthreads();
      double worst = 0.0;
#pragma unroll
      for (int q = 0; q < kWideThreads / 32; ++q) worst = fmax(worst, W.red[1 + q]);
      folded = worst <= 1.0;
    }
    ph.mark(WP_FOLD);
    // reload the original [G0 | a]
    load_block(M, Sb, lds, n, nc);
    __syncthreads();
    if (folded) {
      // E = G0 X - a (in place of a): a 2 x 2 output tile per thread (rows i, i + 1; columns c, c + w/2),
      // four independent chains in flight, each in the reference's k order
      const int wh = (w + 1) >> 1, nh = (n + 1) >> 1;
      for (int t = tid; t < nh * wh; t += kWideThreads) {
        const int ip = t / wh, cp = t - ip * wh;
        const int i0 = 2 * ip, c0 = cp;
        const bool vi = i0 + 1 < n, vc = cp + wh < w;
        const int i1 = vi ? i0 + 1 : i0, c1 = vc ? cp + wh : cp;
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
        const double* g0 = M + i0 * nc;
        const double* g1 = M + i1 * nc;
#pragma unroll 4
        for (int k = 0; k < n; ++k) {
          const double ga = g0[k], gb = g1[k], x0 = X[k * w + c0], x1 = X[k * w + c1];
          a00 = add(a00, mul(ga, x0));
          a01 = add(a01, mul(ga, x1));
          a10 = add(a10, mul(gb, x0));
          a11 = add(a11, mul(gb, x1));
        }
        double* e0 = M + i0 * nc + n;
        double* e1 = M + i1 * nc + n;
        const double b00 = e0[c0], b01 = e0[c1], b10 = e1[c0], b11 = e1[c1];
        e0[c0] = sub(a00, b00);
        if (vc) e0[c1] = sub(a01, b01);
        if (vi) e1[c0] = sub(a10, b10);
        if (vi && vc) e1[c1] = sub(a11, b11);
      }
      __syncthreads();
    }
    if (tid < n) {
      double s = 0.0;
      const double* mrow = M + tid * nc + n;
#pragma unroll 4
      for (int c = 0; c < w; ++c) s = add(s, fabs(mrow[c]));
      double* d = Sb + tid * lds + off_new + tid;
      *d = add(*d, folded ? mul(s, 1.0 + 1e-12) : s);
    }
    // G0 (column-scaled by 1 + r_j when folded) moves right by w
    for (int i = warp; i < n; i += kWideThreads / 32)
      for (int j = lane; j < n; j += 32) {
        const double g = M[i * nc + j];
        Sb[i * lds + w + j] = folded ? mul(g, add(1.0, rr[j])) : g;
      }
    __syncthreads();
    if (tid == 0)
      for (int q = 0; q + 1 < nq; ++q) W.wid[q] = W.wid[q + 1];
    __syncthreads();
    base += w;
    --nq;
  }
}

// The wide horizon kernel: dt_reach (l == 0) or the DT closed loop (l > 0),
// one CTA per sample, persistent over the batch.
template <int RD, int RC>
__global__ void __launch_bounds__(kWideThreads, 1) dt_wide_kernel(const DTParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sd = reinterpret_cast<double*>(smem_raw);
  const int tid = threadIdx.x;
  const int n = P.n, m = P.m, H = P.H, lc = P.l;
  const int n_i = n + lc;
  const int cap = P.window > 0 ? P.window : 1;
  const int nomax = max(n, lc);
  WideSmem W;
  W.nop = P.w_nop;
  W.hw = P.w_hw;
  W.lt = sd;
  W.stages = sd + P.w_o_stage;
  W.relax = sd + P.w_o_relax;
  W.bf0 = sd + P.w_o_bf0;
  double* ms = sd + P.w_o_misc;
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
  int* is = reinterpret_cast<int*>(sd + P.w_o_int);
  W.wid = is;
  W.iv = is + 16;
  W.cnt = is + 32;
  W.lists = reinterpret_cast<unsigned char*>(is + 48);
  W.bars = reinterpret_cast<uint64_t*>(sd + P.w_o_bar);

  const long long lds = P.w_lds;
  double* buf0 = P.wws + static_cast<long long>(blockIdx.x) * P.wws_stride;
  WPhase ph{P.w_phase, clock64(), WP_SETUP};

  for (long long b = blockIdx.x; b < P.B; b += gridDim.x) {
    ph.mark(WP_SETUP);
    const double* act_base = P.actions;
    if (!P.actions_shared && m > 0) act_base += static_cast<size_t>(b) * H * m;
    // ---- X0 and init_symbolic_state (flowpipe_ct.hpp:303-309)
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
    int base = 0, nq = 0;
    auto init_state = [&]() {  // from the box in xlo / xhi
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
      if constexpr (RC > 0) {
        // ---- controller: u_tm = ctl_crown(x_tm, ctl, {}) (neural.hpp:418-424); its
        // generator rows land under x's rows in the same buffer ([x; u] stacking)
        const int rc = wide_certify<RC>(P.ctl, n, lc, n, nullptr, cur + base, lds, nz, nullptr, W.cst,
                                        cur + n * lds + base, lds, W, ph, 0);
        if (rc != WC_OK) {
          status = (rc == WC_PREACT) ? ST_CTL_PREACT : ST_CTL_CERT;
          failed_step = k;
          break;
        }
        if (tid < lc) {
          W.urad[tid] = mul(sub(W.rh[tid], W.rl[tid]), 0.5);
          W.cag[n + tid] = add(W.mid[tid], mul(add(W.rl[tid], W.rh[tid]), 0.5));
        }
        if (tid < n) W.cag[tid] = add(W.cst[tid], 0.0);  // x_tm.c + mid([0,0])
        __syncthreads();
        cin = W.cag;
        frad = W.urad;
      }
      // ---- dynamics / one-step map: certify_tm_input (neural.hpp:342-394), its output written in place at
      // column 0 of the same buffer: output column j depends only on input column base + j >= j, and every
      // column pass of the prepend GEMM has read its input before it writes (one state buffer per CTA)
      const int rc = wide_certify<RD>(P.net, n_i, n, n, u, cur + base, lds, nz, frad, cin, cur, lds, W, ph, 5);
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
        cur[i * lds + nza + j] = (i == j) ? W.radv[i] : 0.0;
      }
      nq += (lc > 0) ? 2 : 1;
      base = 0;
      __syncthreads();
      // ---- fold_overflow (flowpipe_ct.hpp:317-350)
      ph.mark(WP_FOLD);
      wide_fold<8 * RD>(cur, lds, n, base, nq, cap, W, ph);
      ph.mark(WP_BOX);
      // ---- symbolic_box (flowpipe_ct.hpp:413-424)
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
    }
    ph.mark(WP_SETUP);
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
}

}  // namespace rb
