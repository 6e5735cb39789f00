// Fused discrete-time reachability horizon kernel for B200 (sm_100a).
//
// One warp owns one sample (an initial-set sub-box or an MPC candidate) for
// the WHOLE horizon; its symbolic state (c, G0, the windowed generator queue)
// stays in shared memory across steps, so nothing but the final boxes ever
// reaches HBM.  A dedicated producer warp streams the network's weight
// matrices -- the only operand shared across samples -- through a ring of
// shared-memory stages with the bulk-copy (TMA) engine and mbarriers; every
// sample warp of the CTA consumes the same stream, so each weight byte is
// read from L2 once per CTA per step and reused by all of its samples.
//
// Per step each warp runs the reference's dt_reach step (dt_reach.hpp:52-102):
//   certify_tm_input (neural.hpp:342-394) on the symbolic seed:
//     IBP preactivation bounds through the frozen net (neural.hpp:243-257),
//     CROWN backward with shared slopes (neural.hpp:290-335): relaxation +
//     intercept/shift chains, then the dense Lambda.W contraction,
//     the prepended [A|I] layer and the remainder tail;
//   re-seed (dt_reach.hpp:69-92), fold_overflow (flowpipe_ct.hpp:317-350)
//   with a warp-parallel partial-pivot solve (linalg.hpp:96-132), and
//   symbolic_box (flowpipe_ct.hpp:413-424).
// Every floating-point reduction runs in the reference's order with separate
// multiply and add roundings, so the result is bit-identical to the
// reference's scalar C++ (ReLU networks; tanh uses CUDA's libm).
#pragma once

#include "dt_common.cuh"

namespace rb {

constexpr int kMaxLayers = 8;
constexpr int kMaxSplitDims = 16;

struct DevNet {
  int L;
  int dims[kMaxLayers + 1];
  int acts[kMaxLayers];
  long long w_off[kMaxLayers];   // W_l  : dims[l+1] rows x ldw[l]   (row-major, cols = dims[l], zero-padded)
  long long wt_off[kMaxLayers];  // W_l^T: dims[l] rows x ldt[l]     (cols = dims[l+1], zero-padded)
  long long b_off[kMaxLayers];   // b_l padded with zeros to a multiple of 32
  int ldw[kMaxLayers];
  int ldt[kMaxLayers];
  const double* blob;
};

constexpr int kMaxChunks = 96;  // weight-stream chunks per DT step
// shared-memory header: 8 mbarriers, 16 counters, the chunk table
constexpr int kHeaderBytes = (128 + kMaxChunks * 12 + 127) / 128 * 128;

struct DTParams {
  DevNet net;       // the one-step map (DT) or the dynamics network (closed loop)
  DevNet ctl;       // closed loop only: the controller network (l outputs)
  int l;            // control dimension; 0 = open-loop dt_reach
  int B, H, n, m, window, rebuild;
  // per-sample inputs (tube mode) -- or split mode (sub-box from the grid)
  const double* x0_lo;
  const double* x0_hi;
  int split;
  long long part_begin;
  int counts[kMaxSplitDims];
  double sx_lo[kMaxSplitDims];
  double sx_hi[kMaxSplitDims];
  const double* actions;
  int actions_shared;
  int x0_center;    // 1: every sample's X0 = box_from_center(x0_lo[0..n), x0_eps) (interval.hpp:224-235)
  double x0_eps;
  // tube outputs
  double* out_lo;
  double* out_hi;
  int* n_boxes;
  int* failed_step;
  int* status;
  // hull outputs (split mode)
  unsigned long long* hull_lo;  // order keys [H+1][n]
  unsigned long long* hull_hi;
  int* hull_div;                // [H+1]
  int* hull_nan0;               // [H+1][n][2], part-0 NaN rule
  int* hull_nboxes;             // [1]
  unsigned long long* hull_fail_key;  // [1]
  // shared-memory layout (doubles)
  int stage_doubles, nstage, warp_doubles, bias_doubles;
  int o_stA, o_c, o_pre, o_LT, o_R, o_bf0, o_idx;  // hb aliases LT; R only for tanh nets
  int o_aug, ldag, o_cag;       // closed loop: stacked [x; u] TM ((n+l) x ldag) and its centre
  int o_wid;                    // generator block widths (ints)
  int has_tanh;
  int nzs;                      // stA row stride (n * (cap + 2))
  int hp;                       // padded hidden width (32 * CPL)
  int bias_s_off[kMaxLayers];   // per-layer bias offsets in the CTA bias copy
  int bias_s_off_ctl[kMaxLayers];
  // weight stream: chunk table of one DT step (the sequence repeats every step);
  // entries are absolute device addresses (the two networks live in two blobs)
  int n_chunks_step;
  long long ch_off[kMaxChunks];
  unsigned ch_bytes[kMaxChunks];
  // wide family (wide_kernel.cuh): one CTA per sample, symbolic state in global memory
  double* wws;              // per-CTA workspace: two state buffers of w_rows x w_lds
  long long wws_stride;     // doubles per CTA
  int w_lds, w_rows;        // state row stride / rows (n + l)
  int w_nop, w_hw;          // Lambda^T row stride (odd), widest streamed row / unit count
  int w_o_stage, w_o_relax, w_o_bf0, w_o_misc, w_o_int, w_o_bar;  // shared-memory offsets (doubles)
  unsigned long long* w_phase;  // optional per-phase cycle counters (RB_WIDE_PHASE=1), else null
};

enum : int { ST_OK = 0, ST_PREACT = 1, ST_CERT = 2, ST_BOX = 3, ST_CTL_PREACT = 4, ST_CTL_CERT = 5 };

// Weight stream: a ring of shared-memory stages filled by the bulk-copy (TMA)
// engine.  Every sample warp consumes every chunk in the same order; the LAST
// warp to release a stage refills it with the chunk NSTAGE ahead, so no warp
// is dedicated to producing and no warp blocks on a slow sibling to refill.
struct WStream {
  double* stages;
  uint64_t* full;
  int* cnt;
  const long long* ch_off;      // shared-memory copy of the chunk table (device addresses)
  const unsigned* ch_bytes;
  int spc, nstage, stage_doubles, n_chunks_step;
  uint32_t g;
  uint32_t total;
  int sidx = 0;      // g % nstage, tracked incrementally
  uint32_t ph = 0u;  // (g / nstage) & 1
#ifdef RB_PHASE_TIMING
  long long wait_cycles = 0;
#endif
  __device__ __forceinline__ void issue(uint32_t gn, int s) const {
    const int idx = static_cast<int>(gn % static_cast<uint32_t>(n_chunks_step));
    const uint32_t bytes = ch_bytes[idx];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_g2s(stages + static_cast<size_t>(s) * stage_doubles, reinterpret_cast<const double*>(ch_off[idx]), bytes,
             &full[s]);
  }
  // Waits for the current chunk; returns its stage index (the caller forms the
  // pointer from its own shared-memory base so the address space stays known).
  __device__ __forceinline__ int acquire() {
#ifdef RB_PHASE_TIMING
    const long long t0 = clock64();
#endif
    mbar_wait(&full[sidx], ph);
#ifdef RB_PHASE_TIMING
    wait_cycles += clock64() - t0;
#endif
    return sidx;
  }
  __device__ __forceinline__ void release(int lane) {
    __syncwarp();
    if (lane == 0) {
      const int s = sidx;
      int old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(old)
                   : "r"(smem_u32(&cnt[s]))
                   : "memory");
      if (old == spc - 1) {
        cnt[s] = 0;
        const uint32_t gn = g + nstage;
        if (gn < total) issue(gn, s);
      }
    }
    ++g;
    if (++sidx == nstage) {
      sidx = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ int rows_per_chunk(int ld, int stage_doubles) {
  int r = stage_doubles / ld;
  return r < 1 ? 1 : r;
}

// relax_activation (neural.hpp:166-227) for ReLU / tanh; identity never relaxed.
__device__ __forceinline__ void relax(int act, double l, double u, double& s, double& li, double& ui) {
  s = 0.0;
  li = 0.0;
  ui = 0.0;
  if (act == 0) {  // relu
    if (l >= 0.0) {
      s = 1.0;
    } else if (u <= 0.0) {
      s = 0.0;
    } else {
      const double sl = __ddiv_rn(u, sub(u, l));
      s = sl;
      ui = mul(-sl, l);
      li = smin(0.0, smin(mul(-sl, l), sub(u, mul(sl, u))));
    }
  } else {  // tanh
    const double tl = tanh(l), tu = tanh(u);
    const double sl = smin(sub(1.0, mul(tl, tl)), sub(1.0, mul(tu, tu)));
    s = sl;
    double lo = sub(tl, mul(sl, l));
    double hi = lo;
    double g = sub(tu, mul(sl, u));
    lo = smin(lo, g);
    hi = smax(hi, g);
    if (sl < 1.0 && sl > 0.0) {
      const double xs = atanh(__dsqrt_rn(sub(1.0, sl)));
      if (l <= xs && xs <= u) {
        g = sub(tanh(xs), mul(sl, xs));
        lo = smin(lo, g);
        hi = smax(hi, g);
      }
      if (l <= -xs && -xs <= u) {
        g = sub(tanh(-xs), mul(sl, -xs));
        lo = smin(lo, g);
        hi = smax(hi, g);
      }
    }
    const double margin = add(mul(sub(hi, lo), 1e-12), 1e-15);
    li = sub(lo, margin);
    ui = add(hi, margin);
  }
}

__device__ __forceinline__ double act_apply(int act, double x) {
  if (act == 0) return smax(x, 0.0);
  if (act == 1) return tanh(x);
  return x;
}

// split_box (refine.hpp:83-115): part p of the grid, last dimension fastest.
__device__ __forceinline__ void split_edges(const DTParams& P, long long p, int d, double& lo, double& hi) {
  long long q = p;
  for (int e = P.n - 1; e > d; --e) q /= P.counts[e];
  const int k = P.counts[d];
  const int i = static_cast<int>(q % k);
  const double xl = P.sx_lo[d], xh = P.sx_hi[d];
  const double w = sub(xh, xl);
  lo = (i == 0) ? xl : add(xl, mul(w, __ddiv_rn(static_cast<double>(i), static_cast<double>(k))));
  hi = (i + 1 == k) ? xh : add(xl, mul(w, __ddiv_rn(static_cast<double>(i + 1), static_cast<double>(k))));
}


// ---------------------------------------------------------------------------
// Optional phase timing (build with -DRB_PHASE_TIMING): clock64 cycles per
// kernel phase, summed over warps, read back with reach_debug_phase_cycles.
#ifdef RB_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
#define RB_PH(i)                               \
  do {                                         \
    const long long now_ = clock64();          \
    ph_acc[ph_cur] += now_ - ph_last;          \
    ph_last = now_;                            \
    ph_cur = (i);                              \
  } while (0)
#else
#define RB_PH(i) \
  do {           \
  } while (0)
#endif
enum { PH_PREP = 0, PH_IBP = 1, PH_BINIT = 2, PH_CHAIN = 3, PH_GEMM = 4, PH_GEMM0 = 5, PH_TAIL = 6, PH_FOLD = 7,
       PH_BOX = 8, PH_DRAIN = 9 };


// Iterates the set bits of `mask` (CPL words, bit o = unit o) inside rows [r0, r0 + nr),
// calling f(row) in ascending order.  The mask is per sample, so warp-uniform.
template <typename F>
__device__ __forceinline__ void for_each_row(const unsigned* mask, int r0, int nr, F&& f) {
  const int r1 = r0 + nr;
  for (int wi = r0 >> 5; wi * 32 < r1; ++wi) {
    unsigned bits = mask[wi];
    const int lo = wi * 32;
    if (r0 > lo) bits &= ~0u << (r0 - lo);
    if (r1 < lo + 32) bits &= (1u << (r1 - lo)) - 1u;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      f(lo + b);
    }
  }
}

// Ascending rows of [r0, r0 + nr) whose mask bit is set (mask == nullptr: every row).
struct RowIter {
  const unsigned* mask;
  int r0, r1, wi, cur;
  unsigned bits;
  __device__ __forceinline__ RowIter(const unsigned* m, int r0_, int nr) : mask(m), r0(r0_), r1(r0_ + nr) {
    cur = r0_;
    wi = (r0_ >> 5) - 1;
    bits = 0u;
  }
  __device__ __forceinline__ int next() {
    if (!mask) return cur < r1 ? cur++ : -1;
    while (bits == 0u) {
      ++wi;
      if (wi * 32 >= r1) return -1;
      unsigned b = mask[wi];
      const int lo = wi * 32;
      if (r0 > lo) b &= ~0u << (r0 - lo);
      if (r1 < lo + 32) b &= (1u << (r1 - lo)) - 1u;
      bits = b;
    }
    const int b = __ffs(bits) - 1;
    bits &= bits - 1u;
    return wi * 32 + b;
  }
};

// Number of set bits of `mask` below bit x.
__device__ __forceinline__ int popc_below(const unsigned* mask, int x) {
  int c = 0;
  const int w = x >> 5;
  for (int i = 0; i < w; ++i) c += __popc(mask[i]);
  if (x & 31) c += __popc(mask[w] & ((1u << (x & 31)) - 1u));
  return c;
}

// popc_below over a per-layer mask held in registers: the CPL words and their prefix counts are read
// once per layer, so the per-chunk row counts need no shared-memory round trips.
template <int CPL>
struct MaskCount {
  unsigned w[CPL];
  int below[CPL];
  __device__ __forceinline__ explicit MaskCount(const unsigned* mask) {
    int c = 0;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      w[q] = mask[q];
      below[q] = c;
      c += __popc(w[q]);
    }
  }
  // number of set bits below bit x (0 <= x <= 32 * CPL)
  __device__ __forceinline__ int count(int x) const {
    const int q = x >> 5, r = x & 31;
    int c = 0;
#pragma unroll
    for (int k = 0; k < CPL; ++k)
      if (k == q) c = below[k] + (r ? __popc(w[k] & ((1u << r) - 1u)) : 0);
    if (q >= CPL) c = below[CPL - 1] + __popc(w[CPL - 1]);
    return c;
  }
};

// Two-deep software pipeline over the rows of `it`: the operands of the next
// row are loaded before the current row's arithmetic is issued, so shared-
// memory latency hides behind the FP64 work of the previous row.
template <class Ops, class Load, class Comp>
__device__ __forceinline__ void pipelined_rows(RowIter& it, Load&& load, Comp&& comp) {
#if !RB_PIPELINE
  for (int j = it.next(); j >= 0; j = it.next()) {
    Ops A;
    load(j, A);
    comp(j, A);
  }
  return;
#endif
  int ja = it.next();
  if (ja < 0) return;
  Ops A, B;
  load(ja, A);
  for (;;) {
    const int jb = it.next();
    if (jb >= 0) load(jb, B);
    comp(ja, A);
    if (jb < 0) return;
    ja = it.next();
    if (ja >= 0) load(ja, A);
    comp(jb, B);
    if (ja < 0) return;
  }
}

// ---------------------------------------------------------------------------
// Kernel configuration.
#ifndef RB_SAMPLE_WARPS
#define RB_SAMPLE_WARPS 12  // 384 threads: <= 170 registers, no spills (ptxas); smem sets the stage size
#endif
#ifndef RB_MIN_BLOCKS
#define RB_MIN_BLOCKS 1
#endif
constexpr int kSampleWarps = RB_SAMPLE_WARPS;
#ifndef RB_GEMM_UNROLL
#define RB_GEMM_UNROLL 4
#endif
#ifndef RB_IBP_UNROLL
#define RB_IBP_UNROLL 4
#endif
constexpr int kGemmUnroll = RB_GEMM_UNROLL;  // row-loop unroll of the Lambda.W contraction
constexpr int kIbpUnroll = RB_IBP_UNROLL;    // row-loop unroll of the IBP stream
constexpr int kNZG = 2;  // 32-column groups of a generator matrix (<= 64 columns)

// Per-warp scratch of one certification (shared memory).
template <int CPL>
struct CertScratch {
  double* pre;            // per hidden layer, per padded unit: (lo,hi) -> after relax (s, ui) [ReLU]
  double* LT;             // Lambda^T [col][NOP]; also the IBP input buffer and the fold scratch
  double* R;              // tanh relaxation (s, li, ui) per unit
  double* bf0;            // frozen first-layer bias
  unsigned* masks;        // [L-1][2][CPL] active / unstable unit bitmasks
  unsigned char* alists;  // [L-1][HP] compacted active units
};

// ---------------------------------------------------------------------------
// certify_tm_input (neural.hpp:342-394) of one sample, by one warp.
//
// Input TM x = c + A z (+ the zero remainder of a symbolic seed), A = n_i x nz
// in shared memory (row stride lda); rows n_i.. of layer 0 are frozen trailing
// inputs u (freeze_trailing_inputs, neural.hpp:398-413).  Consumes the net's
// weight chunks (W^T of the hidden layers, then W of every layer, top down)
// from the stream even when `done`.  Returns A_out = Lambda . A in registers
// (lane = column j of group g, rows i < n_o) and, on lanes < n_o, the tail
// (mid, rem_lo, rem_hi) of neural.hpp:383-391.
template <int NO, int CPL>
__device__ __forceinline__ void certify(const DevNet& N, const double* bias_s, const int* bias_off, int n_i, int n_o,
                                        const double* u, const double* A, int lda, int nz, const double* c,
                                        const CertScratch<CPL>& S, WStream& ws_in, const double* stages, int SD,
                                        int lane, bool done, double (&aout)[NO][kNZG], double& mid, double& rl,
                                        double& rh, bool& preact_bad, bool& lam_bad) {
  constexpr int NOP = (NO + 1) & ~1;  // Lambda^T row stride (16-byte rows)
  constexpr int HP = 32 * CPL;
  const int L = N.L;
  const int m_frz = N.dims[0] - n_i;  // frozen trailing inputs
  double* LT = S.LT;
  double* hb = S.LT;
  preact_bad = false;
  lam_bad = false;

  // ---- prepend layer IBP (neural.hpp:360-373 + interval.hpp:284-295):
  // pre0_i = sum_j iv_scale(A_ij, [-1,1]) (+ the [0,0] remainder block) + c_i
  if (!done && lane < n_i) {
    double lo = 0.0, hi = 0.0;
    for (int j = 0; j < nz; ++j) {
      const double a = A[lane * lda + j];
      lo = add(lo, (a >= 0.0) ? -a : a);  // a*-1 : a*1
      hi = add(hi, (a >= 0.0) ? a : -a);
    }
    const double cl = c[lane];
#if RB_FUSED
    // fused mode: the IBP input boxes are held in mid / radius form (see ibp_row)
    hb[2 * lane] = cl;
    hb[2 * lane + 1] = hi;
#else
    hb[2 * lane] = add(lo, cl);
    hb[2 * lane + 1] = add(hi, cl);
#endif
  }
  __syncwarp();

  // ---- IBP through the hidden layers (neural.hpp:243-257); output layer skipped
  for (int l = 0; l + 1 < L; ++l) {
    const int width = N.dims[l + 1];
    const int rows = N.dims[l];
    const int ld = N.ldt[l];
    const int act = N.acts[l];
    const double* bias = bias_s + bias_off[l];
    const unsigned* in_mask = S.masks + (l - 1) * 2 * CPL;  // l >= 1: active units of layer l-1
    const unsigned char* in_list = S.alists + (l - 1) * HP;
    double alo[CPL], ahi[CPL], bfold[CPL];
#pragma unroll
    for (int cc = 0; cc < CPL; ++cc) {
      alo[cc] = 0.0;
      ahi[cc] = 0.0;
      bfold[cc] = bias[cc * 32 + lane];
    }
    auto ibp_row = [&](const double* ch, int r0, int j) {
      const double* wrow = ch + (j - r0) * ld + lane;
      const double2 x = *reinterpret_cast<const double2*>(hb + 2 * j);
      double w[CPL], tl[CPL], th[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) w[cc] = wrow[cc * 32];
#if RB_FUSED
      // mid / radius IBP: alo accumulates W.mid, ahi accumulates |W|.rad -- two DFMAs per weight, no
      // endpoint selects (equal to the endpoint form up to rounding)
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        alo[cc] = fma(w[cc], x.x, alo[cc]);
        ahi[cc] = fma(fabs(w[cc]), x.y, ahi[cc]);
      }
      (void)tl;
      (void)th;
      return;
#endif
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const bool pos = w[cc] >= 0.0;
        tl[cc] = mul(w[cc], pos ? x.x : x.y);
        th[cc] = mul(w[cc], pos ? x.y : x.x);
      }
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        alo[cc] = add(alo[cc], tl[cc]);
        ahi[cc] = add(ahi[cc], th[cc]);
      }
    };
    const int rpc = rows_per_chunk(ld, SD);
    int t = 0;
    const MaskCount<CPL> imc(l > 0 ? in_mask : S.masks);
    for (int r0 = 0; r0 < rows; r0 += rpc) {
      const double* ch = stages + ws_in.acquire() * SD;
      const int nr = min(rpc, rows - r0);
      if (!done) {
        if (l > 0) {
          const int t1 = imc.count(r0 + nr);
#pragma unroll kIbpUnroll
          for (; t < t1; ++t) ibp_row(ch, r0, in_list[t]);
        } else {
          const int nx = min(n_i, r0 + nr);
#pragma unroll kIbpUnroll
          for (int j = r0; j < nx; ++j) ibp_row(ch, r0, j);
          // freeze_trailing_inputs (neural.hpp:410): b += W[:, n_i + j] u_j
          for (int r = max(n_i - r0, 0); r < nr; ++r) {
            const double uj = u[r0 + r - n_i];
            const double* wrow = ch + r * ld + lane;
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) bfold[cc] = add(bfold[cc], mul(wrow[cc * 32], uj));
          }
        }
      }
      ws_in.release(lane);
    }
    if (!done) {
      double* pl = S.pre + l * 2 * HP;
      unsigned* am = S.masks + l * 2 * CPL;
      int lbase = 0;
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const int o = cc * 32 + lane;
#if RB_FUSED
        const double pm = alo[cc] + bfold[cc];
        const double plo = pm - ahi[cc];
        const double phi = pm + ahi[cc];
#else
        const double plo = add(alo[cc], bfold[cc]);
        const double phi = add(ahi[cc], bfold[cc]);
#endif
        *reinterpret_cast<double2*>(pl + 2 * o) = make_double2(plo, phi);
        if (l == 0 && m_frz > 0) S.bf0[o] = bfold[cc];
        const bool fin = finite(plo) && finite(phi);
        if (o < width && act != 2 && !fin) preact_bad = true;
        // ReLU slope (neural.hpp:166-227): 1 if lo >= 0 (a [0,0] preactivation is
        // stably active), else 0 if hi <= 0 (inactive), else unstable.  Other acts: dense.
        const bool actv = (o < width) && ((act != 0) || plo >= 0.0 || !(phi <= 0.0));
        const bool unst = (o < width) && ((act != 0) || (plo < 0.0 && phi > 0.0) || !fin);
        const unsigned ma = __ballot_sync(0xffffffffu, actv);
        const unsigned mu = __ballot_sync(0xffffffffu, unst);
        if (lane == 0) {
          am[cc] = ma;
          am[CPL + cc] = mu;
        }
        if (actv) S.alists[l * HP + lbase + __popc(ma & ((1u << lane) - 1u))] = static_cast<unsigned char>(o);
        lbase += __popc(ma);
        alo[cc] = act_apply(act, plo);
        ahi[cc] = act_apply(act, phi);
      }
      __syncwarp();  // every lane is done reading hb
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc)
#if RB_FUSED
        *reinterpret_cast<double2*>(hb + 2 * (cc * 32 + lane)) =
            make_double2(0.5 * (alo[cc] + ahi[cc]), 0.5 * (ahi[cc] - alo[cc]));
#else
        *reinterpret_cast<double2*>(hb + 2 * (cc * 32 + lane)) = make_double2(alo[cc], ahi[cc]);
#endif
      __syncwarp();
    }
  }
  if (!done) preact_bad = __any_sync(0xffffffffu, preact_bad);

  // ---- CROWN backward (neural.hpp:297-327)
  // init: Lambda = I . W_{L-1} = W_{L-1};  b = 0 + I . b_{L-1}
  double blo = 0.0, bup = 0.0;
  {
    const int l = L - 1;
    const int rows = N.dims[l + 1];  // = n_o
    const int ncols = (l == 0) ? n_i : N.dims[l];
    const int ld = N.ldw[l];
    const int rpc = rows_per_chunk(ld, SD);
    for (int r0 = 0; r0 < rows; r0 += rpc) {
      const double* ch = stages + ws_in.acquire() * SD;
      const int nr = min(rpc, rows - r0);
      if (!done) {
        for (int r = 0; r < nr; ++r) {
          const int i = r0 + r;
          for (int j = lane; j < ncols; j += 32) LT[j * NOP + i] = add(0.0, ch[r * ld + j]);
        }
      }
      ws_in.release(lane);
    }
    if (!done && lane < n_o) {
      double bi = bias_s[bias_off[l] + lane];
      if (l == 0 && m_frz > 0) {  // single-layer net: fold the frozen inputs into the bias here
        const double* w = N.blob + N.w_off[0] + static_cast<size_t>(lane) * N.ldw[0];
        for (int j = 0; j < m_frz; ++j) bi = add(bi, mul(w[n_i + j], u[j]));
        S.bf0[lane] = bi;
      }
      blo = add(0.0, bi);
      bup = blo;
    }
    __syncwarp();
  }
  for (int l = L - 2; l >= 0; --l) {
    const int act = N.acts[l];
    const int width = N.dims[l + 1];
    const double* bvec = (l == 0 && m_frz > 0) ? S.bf0 : bias_s + bias_off[l];
    const unsigned* am = S.masks + l * 2 * CPL;
    double* pl = S.pre + l * 2 * HP;
    if (!done) {
      if (act == 0) {
        // ReLU relaxation (parallel): (s, ui) overwrite the preactivation slots; li = 0
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          const int o = cc * 32 + lane;
          const double2 p = *reinterpret_cast<const double2*>(pl + 2 * o);
          double s, li, ui;
          relax(0, p.x, p.y, s, li, ui);
          *reinterpret_cast<double2*>(pl + 2 * o) = make_double2(s, ui);
        }
        __syncwarp();
#if RB_FUSED
        // fused mode: intercepts, slope scaling and the shift Lambda_s . b in ONE lane-parallel pass over
        // this lane's units (the reference sums each row's chain in unit order; here per-lane partial
        // sums and a butterfly reduction -- same terms, a different association)
        {
          double pu[NO], pd[NO], sh[NO];
#pragma unroll
          for (int i = 0; i < NO; ++i) pu[i] = pd[i] = sh[i] = 0.0;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) {
            const int o = cc * 32 + lane;
            if (o < width) {
              const double2 su = *reinterpret_cast<const double2*>(pl + 2 * o);
              const bool unst = (am[CPL + cc] >> lane) & 1u;
              const double bj = bvec[o];
              double* col = LT + o * NOP;
#pragma unroll
              for (int i = 0; i < NOP; i += 2) {
                const double2 v = *reinterpret_cast<const double2*>(col + i);
                const double a0 = v.x, a1 = v.y;
                if (unst) {
                  if (a0 >= 0.0) pu[i] = fma(a0, su.y, pu[i]);
                  else pd[i] = fma(a0, su.y, pd[i]);
                  if (i + 1 < NO) {
                    if (a1 >= 0.0) pu[i + 1] = fma(a1, su.y, pu[i + 1]);
                    else pd[i + 1] = fma(a1, su.y, pd[i + 1]);
                  }
                }
                const double s0 = a0 * su.x, s1 = a1 * su.x;
                *reinterpret_cast<double2*>(col + i) = make_double2(s0, s1);
                sh[i] = fma(s0, bj, sh[i]);
                if (i + 1 < NO) sh[i + 1] = fma(s1, bj, sh[i + 1]);
              }
            }
          }
#pragma unroll
          for (int off = 16; off; off >>= 1)
#pragma unroll
            for (int i = 0; i < NO; ++i) {
              pu[i] += __shfl_xor_sync(0xffffffffu, pu[i], off);
              pd[i] += __shfl_xor_sync(0xffffffffu, pd[i], off);
              sh[i] += __shfl_xor_sync(0xffffffffu, sh[i], off);
            }
#pragma unroll
          for (int i = 0; i < NO; ++i)
            if (lane == i) {
              bup += pu[i] + sh[i];
              blo += pd[i] + sh[i];
            }
          __syncwarp();
        }
        if (false) {
#else
        if (true) {
#endif
        // intercept chains over the unstable units (unscaled Lambda), lane i = row i
        if (lane < n_o) {
          for_each_row(am + CPL, 0, width, [&](int j) {
            const double a = LT[j * NOP + lane];
            const double ui = pl[2 * j + 1];
            if (a >= 0.0) bup = add(bup, mul(a, ui));
            else blo = add(blo, mul(a, ui));
          });
        }
        __syncwarp();
        // slope scaling (parallel over units): Lambda(:, j) *= s_j
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          const int o = cc * 32 + lane;
          const double s = pl[2 * o];
          double* col = LT + o * NOP;
#pragma unroll
          for (int i = 0; i < NOP; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(col + i);
            *reinterpret_cast<double2*>(col + i) = make_double2(mul(v.x, s), mul(v.y, s));
          }
        }
        __syncwarp();
        // shift chain Lambda_s . b (dense; inactive units add +-0), lane i = row i
        if (lane < n_o) {
          double shift = 0.0;
#pragma unroll 8
          for (int j = 0; j < width; ++j) shift = add(shift, mul(LT[j * NOP + lane], bvec[j]));
          blo = add(blo, shift);
          bup = add(bup, shift);
        }
        }  // exact-mode chains
      } else {
        if (act == 1) {
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) {
            const int o = cc * 32 + lane;
            const double2 p = *reinterpret_cast<const double2*>(pl + 2 * o);
            double s, li, ui;
            relax(1, p.x, p.y, s, li, ui);
            S.R[3 * o] = s;
            S.R[3 * o + 1] = li;
            S.R[3 * o + 2] = ui;
          }
          __syncwarp();
        }
        if (lane < n_o) {
          double shift = 0.0;
          if (act == 1) {
            for (int j = 0; j < width; ++j) {
              const double a = LT[j * NOP + lane];
              const double s = S.R[3 * j], li = S.R[3 * j + 1], ui = S.R[3 * j + 2];
              const bool pos = a >= 0.0;
              blo = add(blo, mul(a, pos ? li : ui));
              bup = add(bup, mul(a, pos ? ui : li));
              const double as = mul(a, s);
              LT[j * NOP + lane] = as;
              shift = add(shift, mul(as, bvec[j]));
            }
          } else {
            for (int j = 0; j < width; ++j) shift = add(shift, mul(LT[j * NOP + lane], bvec[j]));
          }
          blo = add(blo, shift);
          bup = add(bup, shift);
        }
      }
      __syncwarp();
    }
    // dense contraction Lambda <- Lambda_s . W_l  (linalg.hpp:53-63, i-k-j order) over the rows
    // k of units with a non-zero slope
    const int ld = N.ldw[l];
    const int rpc = rows_per_chunk(ld, SD);
    const unsigned char* alist = S.alists + l * HP;
    if (l > 0) {
      double acc[NO][CPL];
#pragma unroll
      for (int i = 0; i < NO; ++i)
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) acc[i][cc] = 0.0;
      int t = 0;
      const MaskCount<CPL> amc(am);
      for (int r0 = 0; r0 < width; r0 += rpc) {
        const double* ch = stages + ws_in.acquire() * SD;
        const int nr = min(rpc, width - r0);
        if (!done) {
          const int t1 = amc.count(r0 + nr);
#pragma unroll kGemmUnroll
          for (; t < t1; ++t) {
            const int kk = alist[t];
            const double* lrow = LT + kk * NOP;
            const double* wrow = ch + (kk - r0) * ld + lane;
            double lam[NOP], w[CPL];
#pragma unroll
            for (int i = 0; i < NOP; i += 2) {
              const double2 v = *reinterpret_cast<const double2*>(lrow + i);
              lam[i] = v.x;
              lam[i + 1] = v.y;
            }
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) w[cc] = wrow[cc * 32];
            double tt[NO][CPL];
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
              for (int cc = 0; cc < CPL; ++cc) tt[i][cc] = mul(lam[i], w[cc]);
#pragma unroll
            for (int i = 0; i < NO; ++i)
#pragma unroll
              for (int cc = 0; cc < CPL; ++cc) acc[i][cc] = add(acc[i][cc], tt[i][cc]);
          }
        }
        ws_in.release(lane);
      }
      if (!done) {
        const int ncols = N.dims[l];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc)
#pragma unroll
          for (int i = 0; i < NO; ++i)
            if (i < n_o && cc * 32 + lane < ncols && !finite(acc[i][cc])) lam_bad = true;
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          double* dst = LT + (cc * 32 + lane) * NOP;
#pragma unroll
          for (int i = 0; i < NOP; i += 2)
            *reinterpret_cast<double2*>(dst + i) = make_double2(acc[i][cc], (i + 1 < NO) ? acc[i + 1][cc] : 0.0);
        }
        __syncwarp();
      }
    } else {
      // frozen first layer: only the n_i TM columns survive -- a tiny GEMM
      // (n_o x width) . (width x n_i); lane p owns outputs p and p + 32 of the
      // n_o x n_i grid, each a sequential k chain as the reference's.
      const int npair = n_o * n_i;
      const int p0 = lane, p1 = lane + 32;
      const int i0 = (p0 < npair ? p0 : 0) / n_i, j0 = (p0 < npair ? p0 : 0) % n_i;
      const int i1 = (p1 < npair ? p1 : 0) / n_i, j1 = (p1 < npair ? p1 : 0) % n_i;
      double a0 = 0.0, a1 = 0.0;
      int t = 0;
      const MaskCount<CPL> amc(am);
      for (int r0 = 0; r0 < width; r0 += rpc) {
        const double* ch = stages + ws_in.acquire() * SD;
        const int nr = min(rpc, width - r0);
        if (!done) {
          const int t1 = amc.count(r0 + nr);
#pragma unroll 4
          for (; t < t1; ++t) {
            const int kk = alist[t];
            const double* wrow = ch + (kk - r0) * ld;
            a0 = add(a0, mul(LT[kk * NOP + i0], wrow[j0]));
            a1 = add(a1, mul(LT[kk * NOP + i1], wrow[j1]));
          }
        }
        ws_in.release(lane);
      }
      if (!done) {
        if ((p0 < npair && !finite(a0)) || (p1 < npair && !finite(a1))) lam_bad = true;
        __syncwarp();
        if (p0 < npair) LT[j0 * NOP + i0] = a0;
        if (p1 < npair) LT[j1 * NOP + i1] = a1;
        __syncwarp();
      }
    }
  }
  if (done) return;

  // ---- prepended layer W = [A | I], b = c: shift chain and A_out = Lambda . A
  if (lane < n_o) {
    double shift = 0.0;
    for (int kk = 0; kk < n_i; ++kk) shift = add(shift, mul(LT[kk * NOP + lane], c[kk]));
    blo = add(blo, shift);
    bup = add(bup, shift);
  }
#pragma unroll
  for (int g = 0; g < kNZG; ++g) {
    const int j = g * 32 + lane;
#pragma unroll
    for (int i = 0; i < NO; ++i) aout[i][g] = 0.0;
    if (j < nz) {
      for (int kk = 0; kk < n_i; ++kk) {
        const double akj = A[kk * lda + j];
#pragma unroll
        for (int i = 0; i < NO; ++i) aout[i][g] = mac(aout[i][g], LT[kk * NOP + i], akj);
      }
    }
  }
  // ---- tail (neural.hpp:383-391)
  mid = 0.0;
  rl = 0.0;
  rh = 0.0;
  bool rem_ok = true;
  if (lane < n_o) {
    mid = mul(add(blo, bup), 0.5);
    rl = sub(blo, mid);
    rh = sub(bup, mid);
    rem_ok = finite(rl) && finite(rh);
  }
  lam_bad = !__all_sync(0xffffffffu, rem_ok && !lam_bad);  // reused as "remainder not finite"
}

// ---------------------------------------------------------------------------
// fold_overflow (flowpipe_ct.hpp:317-350) on a symbolic state whose generator
// blocks have widths wid[0..nq) (G0 = stA[:, 0:n], square).  Lane j < n + w
// holds column j of [G0 | oldest block] in registers; pivots and multipliers
// travel by shuffles (partial pivoting, first maximum wins, linalg.hpp:96-132).
template <int NO>
__device__ __forceinline__ void fold_overflow_warp(double* stA, int nzs, int n, int* wid, int& nq, int cap,
                                                   double* scratch, int lane) {
  while (nq > cap) {
    const int w = wid[0];
    const int nc = n + w;
    constexpr int MR = NO;  // rows
    double col[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) col[i] = (lane < nc && i < n) ? stA[i * nzs + lane] : 0.0;
    bool ok = true;
    for (int kk = 0; kk < n; ++kk) {
      int piv = kk;
      double best = 0.0;
#pragma unroll
      for (int i = 0; i < MR; ++i) {
        const double v = fabs(col[i]);
        if (i == kk) best = v;
        if (i > kk && i < n && v > best) {
          best = v;
          piv = i;
        }
      }
      piv = __shfl_sync(0xffffffffu, piv, kk);
      best = __shfl_sync(0xffffffffu, best, kk);
      if (!(best > 1e-12)) {
        ok = false;
        break;
      }
      if (piv != kk) {
        double vk = 0.0, vp = 0.0;
#pragma unroll
        for (int i = 0; i < MR; ++i) {
          if (i == kk) vk = col[i];
          if (i == piv) vp = col[i];
        }
#pragma unroll
        for (int i = 0; i < MR; ++i) {
          if (i == kk) col[i] = vp;
          if (i == piv) col[i] = vk;
        }
      }
      double f[MR];
      double akk = 0.0;
#pragma unroll
      for (int i = 0; i < MR; ++i)
        if (i == kk) akk = col[i];
#if RB_FUSED
      // fused mode: one reciprocal per pivot instead of a division per row
      const double rak = 1.0 / akk;
#pragma unroll
      for (int i = 0; i < MR; ++i) f[i] = (i > kk && i < n) ? col[i] * rak : 0.0;
#else
#pragma unroll
      for (int i = 0; i < MR; ++i) f[i] = (i > kk && i < n) ? __ddiv_rn(col[i], akk) : 0.0;
#endif
#pragma unroll
      for (int i = 0; i < MR; ++i) f[i] = __shfl_sync(0xffffffffu, f[i], kk);
      double mk = 0.0;
#pragma unroll
      for (int i = 0; i < MR; ++i)
        if (i == kk) mk = col[i];
      if (lane < nc && lane >= kk) {
#pragma unroll
        for (int i = 0; i < MR; ++i)
          if (i > kk && i < n) col[i] = sub(col[i], mul(f[i], mk));
      }
    }
    bool folded = false;
    int off_new = n;  // column offset of the newest block
    for (int q = 0; q + 1 < nq; ++q) off_new += wid[q];
    double* newest = stA + off_new;
    double* M = scratch;        // [n][nc] eliminated [U | B']
    double* X = M + n * nc;     // [n][w]
    double* E = X + n * w;      // [n][w]
    double* rr = E + n * w;     // [n]
    if (ok) {
      if (lane < nc)
#pragma unroll
        for (int i = 0; i < MR; ++i)
          if (i < n) M[i * nc + lane] = col[i];
      __syncwarp();
      if (lane >= n && lane < nc) {  // back substitution, lane n+j owns RHS column j
        const int jc = lane - n;
        double x[MR];
#pragma unroll
        for (int i = MR - 1; i >= 0; --i) {
          if (i < n) {
            double a = col[i];
#pragma unroll
            for (int kk = i + 1; kk < MR; ++kk)
              if (kk < n) a = sub(a, mul(M[i * nc + kk], x[kk]));
            x[i] = __ddiv_rn(a, M[i * nc + i]);
            X[i * w + jc] = x[i];
          } else {
            x[i] = 0.0;
          }
        }
      }
      __syncwarp();
      if (lane < n) {
        double s = 0.0;
        for (int j = 0; j < w; ++j) s = add(s, fabs(X[lane * w + j]));
        rr[lane] = mul(s, 1.0 + 1e-12);
      }
      __syncwarp();
      double worst = 0.0;
      for (int j = 0; j < n; ++j) worst = smax(worst, rr[j]);
      if (worst <= 1.0) {
        // residual e = G0 X - a, then scale G0 columns, box e into the newest block
        if (lane < w) {
          for (int i = 0; i < n; ++i) {
            double e = 0.0;
            for (int kk = 0; kk < n; ++kk) e = add(e, mul(stA[i * nzs + kk], X[kk * w + lane]));
            E[i * w + lane] = sub(e, stA[i * nzs + n + lane]);
          }
        }
        __syncwarp();
        if (lane < n) {
          const double sc = add(1.0, rr[lane]);
          for (int i = 0; i < n; ++i) stA[i * nzs + lane] = mul(stA[i * nzs + lane], sc);
          double s = 0.0;
          for (int j = 0; j < w; ++j) s = add(s, fabs(E[lane * w + j]));
          newest[lane * nzs + lane] = add(newest[lane * nzs + lane], mul(s, 1.0 + 1e-12));
        }
        folded = true;
      }
    }
    if (!folded && lane < n) {
      double s = 0.0;
      for (int j = 0; j < w; ++j) s = add(s, fabs(stA[lane * nzs + n + j]));
      newest[lane * nzs + lane] = add(newest[lane * nzs + lane], s);
    }
    __syncwarp();
    // pop the oldest block: columns [n + w, off_end) -> [n, off_end - w)
    const int span = off_new + n - (n + w);  // remaining queue columns (newest block is n wide)
    for (int i = 0; i < n; ++i) {
      for (int j0 = 0; j0 < span; j0 += 32) {
        const int j = j0 + lane;
        const double v = (j < span) ? stA[i * nzs + n + w + j] : 0.0;
        __syncwarp();
        if (j < span) stA[i * nzs + n + j] = v;
        __syncwarp();
      }
    }
    if (lane == 0)
      for (int q = 0; q + 1 < nq; ++q) wid[q] = wid[q + 1];
    __syncwarp();
    --nq;
  }
}

// symbolic_box (flowpipe_ct.hpp:413-424): lane i < n returns box dim i.
__device__ __forceinline__ bool symbolic_box_warp(const double* stA, int nzs, int n, const int* wid, int nq,
                                                  const double* cc, int lane, double& lo, double& hi) {
  lo = 0.0;
  hi = 0.0;
  bool fin = true;
  if (lane < n) {
    double r = 0.0;
    for (int j = 0; j < n; ++j) r = add(r, fabs(stA[lane * nzs + j]));
    int off = n;
    for (int q = 0; q < nq; ++q) {
      double s = 0.0;
      for (int j = 0; j < wid[q]; ++j) s = add(s, fabs(stA[lane * nzs + off + j]));
      r = add(r, s);
      off += wid[q];
    }
    const double c = cc[lane];
    lo = sub(c, r);
    hi = add(c, r);
    fin = finite(lo) && finite(hi);
  }
  return __all_sync(0xffffffffu, fin);
}

// ---------------------------------------------------------------------------
// The horizon kernel: dt_reach (l == 0, dt_reach.hpp:41-104) or the DT closed
// loop (l > 0: controller certification + [x; u] stacking as cl_reach,
// closed_loop.hpp:118-153, then the dynamics certification), one warp per
// sample for the whole horizon, weights streamed through the TMA ring.
template <int NO, int CPL>
__global__ void __launch_bounds__(kSampleWarps * 32, RB_MIN_BLOCKS) dt_horizon_kernel(const DTParams P) {
  constexpr int HP = 32 * CPL;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int spc = blockDim.x / 32;
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  int* cnt = reinterpret_cast<int*>(smem_raw + 64);
  long long* tab_off = reinterpret_cast<long long*>(smem_raw + 128);          // [kMaxChunks]
  unsigned* tab_bytes = reinterpret_cast<unsigned*>(tab_off + kMaxChunks);   // [kMaxChunks]
  double* stages = reinterpret_cast<double*>(smem_raw + kHeaderBytes);
  const int SD = P.stage_doubles;
  double* bias_s = stages + static_cast<size_t>(P.nstage) * SD;
  double* wbase = bias_s + P.bias_doubles;

  const DevNet& N = P.net;
  const int n = P.n, m = P.m, H = P.H, l_ctl = P.l;
  const int cap = P.window > 0 ? P.window : 1;
  const uint32_t total_chunks = static_cast<uint32_t>(P.n_chunks_step) * static_cast<uint32_t>(H);

  for (int i = threadIdx.x; i < P.n_chunks_step; i += blockDim.x) {
    tab_off[i] = P.ch_off[i];
    tab_bytes[i] = P.ch_bytes[i];
  }
  WStream ws_in{stages, full, cnt, tab_off, tab_bytes, spc, P.nstage, SD, P.n_chunks_step, 0u, total_chunks};
  if (threadIdx.x == 0) {
    for (int s = 0; s < P.nstage; ++s) {
      mbar_init(&full[s], 1);
      cnt[s] = 0;
    }
    fence_mbar_init();
  }
  for (int l = 0; l < N.L; ++l) {  // CTA copy of every layer's (padded) bias
    const int cnt_b = (l + 1 < N.L) ? HP : ((N.dims[l + 1] + 1) & ~1);
    for (int i = threadIdx.x; i < cnt_b; i += blockDim.x) bias_s[P.bias_s_off[l] + i] = N.blob[N.b_off[l] + i];
  }
  if (l_ctl > 0)
    for (int l = 0; l < P.ctl.L; ++l) {
      const int cnt_b = (l + 1 < P.ctl.L) ? HP : ((P.ctl.dims[l + 1] + 1) & ~1);
      for (int i = threadIdx.x; i < cnt_b; i += blockDim.x)
        bias_s[P.bias_s_off_ctl[l] + i] = P.ctl.blob[P.ctl.b_off[l] + i];
    }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < P.nstage && static_cast<uint32_t>(s) < total_chunks; ++s) ws_in.issue(s, s);

  // ------------------------------------------------------------ per-warp sample
  const long long b = static_cast<long long>(blockIdx.x) * spc + warp;
  const bool valid = b < P.B;
  double* ws = wbase + static_cast<size_t>(warp) * P.warp_doubles;
  double* stA = ws + P.o_stA;  // n x nzs: [G0 | Q1 .. Qnq | (fresh)]
  double* cc = ws + P.o_c;     // n
  int* wid = reinterpret_cast<int*>(ws + P.o_wid);
  CertScratch<CPL> S{ws + P.o_pre, ws + P.o_LT, ws + P.o_R, ws + P.o_bf0, reinterpret_cast<unsigned*>(ws + P.o_idx),
                     nullptr};
  S.alists = reinterpret_cast<unsigned char*>(S.masks + (max(N.L, P.ctl.L) - 1) * 2 * CPL);
  double* AG = ws + P.o_aug;   // closed loop: stacked (n+l) x ldag
  double* cag = ws + P.o_cag;  // its centre
  const int nzs = P.nzs, ldag = P.ldag;

  const double* act_base = P.actions;
  if (!P.actions_shared && m > 0) act_base += static_cast<size_t>(valid ? b : 0) * H * m;

  // ---- X0 and init_symbolic_state (flowpipe_ct.hpp:303-309)
  double x_lo = 0.0, x_hi = 0.0;
  if (lane < n && valid) {
    if (P.split) {
      split_edges(P, P.part_begin + b, lane, x_lo, x_hi);
    } else if (P.x0_center) {
      const double c = P.x0_lo[lane];
      x_lo = sub(c, P.x0_eps);
      x_hi = add(c, P.x0_eps);
    } else {
      x_lo = P.x0_lo[b * n + lane];
      x_hi = P.x0_hi[b * n + lane];
    }
  }
  auto emit_box = [&](int k, double lo, double hi, bool fin) {
    if (!valid || lane >= n) return;
    if (!P.split) {
      const size_t o = (static_cast<size_t>(b) * (H + 1) + k) * n + lane;
      P.out_lo[o] = lo;
      P.out_hi[o] = hi;
    } else {
      if (lo == lo) atomicMin(&P.hull_lo[k * n + lane], order_key(lo));
      if (hi == hi) atomicMax(&P.hull_hi[k * n + lane], order_key(hi));
      if (P.part_begin + b == 0) {
        if (lo != lo) P.hull_nan0[(k * n + lane) * 2 + 0] = 1;
        if (hi != hi) P.hull_nan0[(k * n + lane) * 2 + 1] = 1;
      }
      if (!fin) atomicOr(&P.hull_div[k], 1);
    }
  };
  auto init_state = [&](double lo, double hi) {
    if (lane < n) {
      cc[lane] = mul(add(lo, hi), 0.5);
      const double rad = mul(sub(hi, lo), 0.5);
      for (int j = 0; j < n; ++j) stA[lane * nzs + j] = (j == lane) ? rad : 0.0;
    }
    __syncwarp();
  };
  emit_box(0, x_lo, x_hi, finite(x_lo) && finite(x_hi));
  init_state(x_lo, x_hi);
  int nq = 0;
  int status = ST_OK, failed_step = -1, nboxes = 1;
  bool done = !valid;

  for (int k = 0; k < H; ++k) {
    const double* u = act_base + static_cast<size_t>(k) * m;
    int nz = n;
    for (int q = 0; q < nq; ++q) nz += wid[q];
    double aout[NO][kNZG];
    double mid, rl, rh;
    bool preact_bad, rem_bad;
    const double* Ain = stA;
    int lda = nzs, nz_in = nz, n_i = n;
    const double* cin = cc;

    if (l_ctl > 0) {
      // ---- controller: u_tm = ctl_crown(x_tm, ctl, {}) (neural.hpp:418-424)
      certify<NO, CPL>(P.ctl, bias_s, P.bias_s_off_ctl, n, l_ctl, nullptr, stA, nzs, nz, cc, S, ws_in, stages, SD,
                       lane, done, aout, mid, rl, rh, preact_bad, rem_bad);
      if (!done && (preact_bad || rem_bad)) {  // cl_reach's controller failures (closed_loop.hpp:106-115)
        status = preact_bad ? ST_CTL_PREACT : ST_CTL_CERT;
        failed_step = k;
        done = true;
      }
      if (!done) {
        // stack [x; u] over the shared variables (closed_loop.hpp:118-153): x rows keep their
        // columns, u rows take the certified control map; fresh block diag(0.., rad(u.rem))
        const int w_new = n + l_ctl;
        for (int i = 0; i < n; ++i)
          for (int j = lane; j < nz + w_new; j += 32) AG[i * ldag + j] = (j < nz) ? stA[i * nzs + j] : 0.0;
#pragma unroll
        for (int g = 0; g < kNZG; ++g) {
          const int j = g * 32 + lane;
          if (j < nz)
#pragma unroll
            for (int i = 0; i < NO; ++i)
              if (i < l_ctl) AG[(n + i) * ldag + j] = aout[i][g];
        }
        const double urad = mul(sub(rh, rl), 0.5);
        const double umid = add(mid, mul(add(rl, rh), 0.5));
        for (int i = 0; i < l_ctl; ++i) {
          const double ri = __shfl_sync(0xffffffffu, urad, i);
          const double mi = __shfl_sync(0xffffffffu, umid, i);
          for (int j = lane; j < w_new; j += 32) AG[(n + i) * ldag + nz + j] = (j == n + i) ? ri : 0.0;
          if (lane == 0) cag[n + i] = mi;
        }
        if (lane < n) cag[lane] = add(cc[lane], 0.0);  // x_tm.c + mid([0,0])
        __syncwarp();
        Ain = AG;
        lda = ldag;
        nz_in = nz + w_new;
        n_i = n + l_ctl;
        cin = cag;
      } else {
        nz_in = nz + n + l_ctl;
      }
    }

    // ---- dynamics / one-step map: certify_tm_input (neural.hpp:342-394)
    certify<NO, CPL>(N, bias_s, P.bias_s_off, n_i, n, u, Ain, lda, nz_in, cin, S, ws_in, stages, SD, lane, done, aout,
                     mid, rl, rh, preact_bad, rem_bad);
    if (done) continue;  // keep draining the weight stream in lockstep
    if (preact_bad || rem_bad) {  // dt_reach.hpp:58-67
      status = preact_bad ? ST_PREACT : ST_CERT;
      failed_step = k;
      done = true;
      continue;
    }
    __syncwarp();
    // ---- re-seed (dt_reach.hpp:69-92): c' = c + mid(rem), blocks <- A_out, fresh = diag(rad(rem))
#pragma unroll
    for (int g = 0; g < kNZG; ++g) {
      const int j = g * 32 + lane;
      if (j < nz_in)
#pragma unroll
        for (int i = 0; i < NO; ++i)
          if (i < n) stA[i * nzs + j] = aout[i][g];
    }
    if (lane < n) {
      cc[lane] = add(mid, mul(add(rl, rh), 0.5));
      const double rad = mul(sub(rh, rl), 0.5);
      for (int j = 0; j < n; ++j) stA[lane * nzs + nz_in + j] = (j == lane) ? rad : 0.0;
    }
    if (lane == 0) {
      if (l_ctl > 0) wid[nq++] = n + l_ctl;
      wid[nq++] = n;
    }
    nq = __shfl_sync(0xffffffffu, nq, 0);
    __syncwarp();

    // ---- fold_overflow (flowpipe_ct.hpp:317-350)
    fold_overflow_warp<NO>(stA, nzs, n, wid, nq, cap, S.LT, lane);

    // ---- symbolic_box (flowpipe_ct.hpp:413-424)
    double lo, hi;
    const bool fin = symbolic_box_warp(stA, nzs, n, wid, nq, cc, lane, lo, hi);
    emit_box(k + 1, lo, hi, fin);
    nboxes = k + 2;
    if (!fin) {
      status = ST_BOX;
      failed_step = k;
      done = true;
      continue;
    }
    __syncwarp();
    if (P.rebuild) {
      init_state(lo, hi);
      nq = 0;
    }
  }

  if (!valid) return;
  if (!P.split) {
    if (lane == 0) {
      P.n_boxes[b] = nboxes;
      P.failed_step[b] = failed_step;
      P.status[b] = status;
    }
  } else if (lane == 0) {
    atomicMin(P.hull_nboxes, nboxes);
    if (status != ST_OK) {
      const unsigned long long key =
          (static_cast<unsigned long long>(failed_step >= 0 ? failed_step : nboxes) << 40) |
          (static_cast<unsigned long long>(P.part_begin + b) << 8) | static_cast<unsigned long long>(status & 0xff);
      atomicMin(P.hull_fail_key, key);
    }
  }
}

// Converts the hull order keys back to doubles, applying the part-0 NaN rule.
static __global__ void hull_finalize_kernel(const unsigned long long* klo, const unsigned long long* khi, const int* nan0,
                                     int count, double* lo, double* hi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  lo[t] = nan0[2 * t] ? __longlong_as_double(0x7ff8000000000000ll) : from_order_key(klo[t]);
  hi[t] = nan0[2 * t + 1] ? __longlong_as_double(0x7ff8000000000000ll) : from_order_key(khi[t]);
}

}  // namespace rb
