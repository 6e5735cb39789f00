// Continuous-time closed-loop reachability kernels for B200 (sm_100a):
// cl_reach (closed_loop.hpp:76-182) with the quadrotor plant augmented by
// udot = 0 rows (make_augmented_field, fields.hpp:96-128; quadrotor_ode,
// systems.hpp:22-64) under a neural (tanh / ReLU) controller.
//
// ct_reach (flowpipe_ct.hpp:428-458) of the analytic fields of fields.hpp
// (zero, diagonal-linear, rotation, quadrotor with a held input) runs the same
// flow kernel alone, with a square G0 and the G0^-1 Q fold.
//
// One warp owns one sub-box.  Per control interval the host launches
//   ct_ctl_kernel   controller certification ctl_crown (neural.hpp:418-424,
//                   certify_tm_input :342-394) on the boundary state TM, the
//                   [x; u] stacking of closed_loop.hpp:122-153 and the hull
//                   fold (flowpipe_ct.hpp:317-350, non-square G0 branch);
//   ct_flow_kernel  k_atomic validated Taylor-model flowpipe steps:
//                   poly_picard (flowpipe_ct.hpp:126-139), remainder_picard
//                   with enlarge / shrink / exact endpoint (:144-276),
//                   tm_eval_interval (taylor_model.hpp:73-97) and
//                   symbolic_step (flowpipe_ct.hpp:378-409).
// The symbolic state (c, [G0 | Q1..Qnq]) of every sub-box stays in HBM
// between the two launches; inside a launch it lives in shared memory.
//
// TMExpr rows (taylor_model.hpp:197-238) are lane-strided in shared memory:
// lane L owns generator columns L, L+32 (, L+64) of az and bz, so every
// TMExpr operation (products with excess folding, integration) is a per-lane
// FP64 update of <= 3 coefficient slots plus warp-uniform scalar interval
// arithmetic; the abs-sums the remainder bounds need (abs_z / abs_b) are
// butterfly shuffle reductions, computed once when a row is produced and
// cached next to it.  Lanes only ever touch their own coefficient slots, so
// the algebra needs no warp barriers.  sin / cos / reciprocal / scalar
// products are scalar multiples of their operand's coefficients and stay
// "views" (no storage, no coefficient pass).  The field itself is a short
// program (kQuadTape) run by one interpreter loop, which keeps the kernel's
// code inside the instruction cache.
//
// Numerics: the reference's operation order inside every TMExpr operation;
// the abs-sums are tree reductions (the reference sums sequentially) and libm
// is CUDA's (sin / cos / tanh), so results agree with the reference to
// rounding (tests: <= 1e-9 relative), not bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "dt_common.cuh"
#include "dt_kernel.cuh"

namespace rb {
namespace ct {

constexpr int NX = 12;      // quadrotor state
constexpr int NA = 16;      // augmented (x, u)
constexpr int NZP = 80;     // generator columns per row (cl_reach: n + window (n + l) <= 76; ct_reach: n (window + 2) <= 80)
constexpr int NZC = (NZP + 31) / 32;  // generator slots per lane (lane + 32 k)
constexpr int kMaxCtlW = 128;  // widest controller layer (and input dim)
constexpr int LDX = NZP + 1;

// REACH_TUBE_* codes
enum : int { CT_OK = 0, CT_CTL_FAILED = 4, CT_CTL_DIVERGED = 5, CT_REMAINDER = 6, CT_PICARD = 7, CT_TME_INV = 8,
             CT_BOX = 3, CT_OTHER = 99 };

// One operation of a field program (see quad / rotation / ... programs built by
// the host, ct_capi.cu): dst / a / b are slot indices, b a constant index for
// SCALE / SUBK / CONST.
struct TOp {
  unsigned char code, dst, a, b;
};
constexpr int kMaxKc = 24;
// Every field program lives in constant memory (uploaded once per device by
// the host, ct_capi.cu): the dispatch reads a provably warp-uniform opcode, so
// the shuffles inside the operations need no divergence handling.
constexpr int kProgCap = 1024;
__constant__ TOp kProgs[kProgCap];

struct CTParams {
  int B, n, l, K, window, order, refine, maxe, intervalize, ref_dim, ci, ctl_steps;
  int na;      // rows of the flowed state: n + l (cl_reach) or n (ct_reach)
  int bw;      // width of a queue block: na in both drivers
  int square;  // 1: G0 is na x na (ct_reach) -> the G0^-1 Q fold; 0: the hull fold
  int ct;      // 1: ct_reach -- no controller; the first launch builds the state from X0
  double h, eps, enl;
  double prm[8];
  double kc[kMaxKc];         // constants of the field program
  int prog;                  // offset of the field program in kProgs
  int fast_prog;             // scalar-only replays: 0 interpreted, 1 / 2 quad_fast<false / true>
  signed char bzsrc[16];     // Picard bz row of row i: -1 own storage, -2 the zero row, j >= 0 the seed row j
  DevNet ctl;
  const double* y_ref;  // device [ctl_steps][ref_dim]
  // initial boxes: batch (x0_lo/hi [B][n]) or split of one box
  const double* x0_lo;
  const double* x0_hi;
  int split;
  long long part_begin;
  int counts[kMaxSplitDims];
  double sx_lo[kMaxSplitDims];
  double sx_hi[kMaxSplitDims];
  // device-resident symbolic state
  double* st_c;  // [B][NA]
  double* st_M;  // [B][NA][NZP]
  int* st_meta;  // [B][4]: nq, status, failed_step, n_boxes
  unsigned char* side;  // [B][kSideBytes]: the compact layout's interval rows + replay cache
  // outputs
  int T;  // boxes per tube (1 + ctl_steps * K)
  double* out_lo;
  double* out_hi;
  int* n_boxes;
  int* failed_step;
  int* status;
  unsigned long long* hull_lo;
  unsigned long long* hull_hi;
  int* hull_div;
  int* hull_nan0;
  int* hull_nboxes;
  unsigned long long* hull_fail_key;
};

// ---------------------------------------------------------------------------
// Interval helpers (interval.hpp:60-94), round to nearest.
struct Iv {
  double lo, hi;
};
__device__ __forceinline__ Iv iadd(Iv a, Iv b) { return Iv{a.lo + b.lo, a.hi + b.hi}; }
__device__ __forceinline__ Iv isub(Iv a, Iv b) { return Iv{a.lo - b.hi, a.hi - b.lo}; }
__device__ __forceinline__ Iv imul(Iv a, Iv b) {
  const double p1 = a.lo * b.lo, p2 = a.lo * b.hi, p3 = a.hi * b.lo, p4 = a.hi * b.hi;
  return Iv{smin(smin(p1, p2), smin(p3, p4)), smax(smax(p1, p2), smax(p3, p4))};
}
// iv_mul({0, H}, {t, t}): the four products are pairwise identical, so
// min(min(p1,p2),min(p3,p4)) = min(0*t, H*t) bit for bit (NaN cases included).
__device__ __forceinline__ Iv imul_0h(double H, double t) {
  const double p1 = 0.0 * t, p3 = H * t;
  return Iv{smin(p1, p3), smax(p1, p3)};
}
__device__ __forceinline__ Iv iscale(double a, Iv x) {
  return (a >= 0.0) ? Iv{a * x.lo, a * x.hi} : Iv{a * x.hi, a * x.lo};
}
__device__ __forceinline__ bool ifin(Iv x) { return isfinite(x.lo) && isfinite(x.hi); }

// Butterfly sums over the warp (identical result on every lane).
__device__ __forceinline__ void wsum2(double& a, double& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}
__device__ __forceinline__ void wsum4(double& a, double& b, double& c, double& d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
}
// Sixteen butterfly sums at once (a transposed reduction): lane L returns
// the sum of v[row_of_wsum16(L)] over the warp.  Every level adds the same
// lane pairs as wsum's butterfly, so each sum is bit-identical to wsum(v[r]);
// 16 + 8 + 4 + 2 + 1 + 1 shuffles instead of 16 x 5.
__device__ __forceinline__ int row_of_wsum16(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}
__device__ __forceinline__ double wsum16_rows(double (&v)[16], int lane) {
#pragma unroll
  for (int o = 16, n = 8; o > 1; o >>= 1, n >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < n) {
        const double got = __shfl_xor_sync(0xffffffffu, up ? v[k] : v[k + n], o);
        v[k] = (up ? v[k + n] : v[k]) + got;
      }
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
__device__ __forceinline__ double wsum(double a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// ---------------------------------------------------------------------------
// TMExpr rows as slots.  A slot is a row of the field evaluation: its
// warp-uniform scalars (centre, time coefficient, remainder, the cached
// abs-sums) plus the shared-memory rows of its az / bz coefficients.
//   P0..      the Picard iterate p_k: az aliases the seed rows S (poly_picard
//             never changes the z columns: g = seed + Int f adds only tau
//             terms); bz in an own row, or aliased (CTParams::bzsrc): a row
//             whose derivative is a copy of P_j has bz = S_j, one whose
//             derivative is 0 has bz = 0;
//   T0..3     full temporaries;
//   V0..9     views: rows whose coefficients are a scalar multiple of another
//             row's (sin / cos linearizations, scalar products, reciprocals,
//             taylor_model.hpp:284-295, 364-425), az = base.az * s, so they
//             cost no coefficient storage and no coefficient pass;
//   C0..3     constant rows (tme_const of a held input, fields.hpp:28).
constexpr int NTF = 4;
constexpr int NV = 10;
constexpr int kFieldCache = 64;  // program entries (before OP_END) a field program may have (FlowSmem::fc)
constexpr int NCST = 4;
constexpr int SLOT_T = NA;
constexpr int SLOT_V = NA + NTF;
constexpr int SLOT_C = SLOT_V + NV;
constexpr int NSLOT = SLOT_C + NCST;

struct Slot {
  double c, at, rlo, rhi;
  double sz, sb;  // abs_z / abs_b (taylor_model.hpp:213-224) of the row's coefficients
  double s1, s2;  // view scales (1, 1 for a stored row)
  int az, bz;     // coefficient rows: offsets (doubles) into FlowSmem::coef()
  int view, pad;
};

// Shared memory of one sub-box: this fixed part, then the coefficient rows
//   S [na][NZP] | zero row | own Picard bz rows | Taz [NTF][NZP] | Tbz [NTF][NZP]
// (cl_reach: 25.6 KB -> 8 sub-boxes per SM).  The Picard bz / temporary rows
// double as the scratch of the square fold.
struct __align__(128) FlowSmem {
  double sc[NA];   // seed centre
  double ssz[NA];  // abs_z of the seed rows
  double ec[NA];   // endpoint centre
  double kc[kMaxKc];
  int pbz[NA];     // Picard bz row offset of row i
  int own[NA];     // row i owns its bz row
  int wid[8];      // queue block widths (square fold)
  int na, off_zero, off_pbz, off_taz, off_tbz, pad;
  Slot D[NSLOT];   // the compact layout keeps D[0, NA) only: the P slots
  // full layout only (the compact layout keeps these in HBM, CTParams::side)
  Iv erem_s[NA], i0_s[NA], i1_s[NA], nx_s[NA];
  double2 fc_s[kFieldCache];  // per program entry: the result's (abs_z, abs_b) / a consumer's replay sum
};
static_assert(sizeof(FlowSmem) % 128 == 0, "coefficient rows start on a 128-byte line: a warp's 256-byte row segment is two smem wavefronts, not three");
// The compact layout (cl_reach under the compiled quadrotor program, ct_flow_kernel<false, true>): the
// header ends after the P slots, the rows are kRowC = 76 columns (n + window (n + l) <= 76 for window
// <= 4) and there is no zero row: 22.1 KB per sub-box -> 10 sub-boxes per SM instead of 8.
constexpr int kRowC = NX + 4 * NA;
constexpr int kNoRow = -(1 << 20);  // "the zero row" in the compact layout: reads give 0
constexpr size_t kCompactHdr = (offsetof(FlowSmem, D) + NA * sizeof(Slot) + 127) / 128 * 128;
template <bool CMP>
__device__ __forceinline__ double* flow_coef(FlowSmem& W) {
  return reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(&W) + (CMP ? kCompactHdr : sizeof(FlowSmem)));
}
// Per-step interval rows and the replay cache: in shared memory (full layout) or in the sub-box's HBM
// block (compact layout; kSideBytes per sub-box).
struct Side {
  Iv *erem, *i0, *i1, *nx;
  double2* fc;
};
constexpr size_t kSideBytes = 4 * NA * sizeof(Iv) + kFieldCache * sizeof(double2);

struct Lane {
  int lane;
  double h;
  bool act[NZC];  // slot lane + 32 k < nz
};

// poly_range (taylor_model.hpp:227-235) from the cached sums.
__device__ __forceinline__ Iv poly_range(double c, double sz, double at, double sb, double h) {
  Iv r{c - sz, c + sz};
  r = iadd(r, imul_0h(h, at));
  const double br = sb * h;
  return iadd(r, Iv{-br, br});
}

// An operand's coefficient rows, read once per operation into registers (the
// coefficient stores of the operation could alias the descriptor otherwise).
// A view of a view (1/cos) carries s1*s2 as one scale: one rounding instead of
// the reference's two, a <= 1 ulp difference inside the stated tolerance.
struct Opnd {
  const double* az;
  const double* bz;
  double s;
  bool view;
};
__device__ __forceinline__ Opnd opnd(const double* coef, const Slot& d) {
  return Opnd{coef + d.az, coef + d.bz, d.s1 * d.s2, d.view != 0};
}
// Branch-free: a stored row carries s = 1 (x * 1.0 == x exactly), so every operand is scaled and the
// per-element view test (9 % of the stall samples, the warp-uniform branch) disappears.
__device__ __forceinline__ void fetch(const Opnd& d, int j, double& a, double& b) {
  a = d.az[j] * d.s;
  b = d.bz[j] * d.s;
}

__device__ __forceinline__ void set_scalars(Slot& r, double c, double at, Iv rem, double sz, double sb) {
  r.c = c;
  r.at = at;
  r.rlo = rem.lo;
  r.rhi = rem.hi;
  r.sz = sz;
  r.sb = sb;
}

// ---- field programs ------------------------------------------------------------
// MUL / ADD / SUB: TMExpr products and sums (taylor_model.hpp:245-360);
// SUBK: TM - s; SCALE: TM * s (a view); SIN / COS / INV: linearizations
// (views); COPY: materialize a view into a temporary; CONST: tme_const(kc);
// CONS i: hand dx_i to the consumer (CONS0: dx_i = 0).
enum : unsigned char {
  OP_MUL, OP_ADD, OP_SUB, OP_SUBK, OP_SCALE, OP_SIN, OP_COS, OP_INV, OP_CONS, OP_CONS0, OP_COPY, OP_CONST, OP_END,
  OP_MUL2  // two independent products: this op (dst = a * b) and the next program entry, one interleaved pass
};
// Between the last Picard iteration and the endpoint the field is evaluated on
// the same Picard iterate p_k with different remainder candidates only
// (remainder_picard's enlarge / shrink replays and the exact endpoint,
// flowpipe_ct.hpp:144-263).  No coefficient of any intermediate row depends on
// a remainder, so the first replay of a step (MODE_REPLAY) runs the full
// coefficient passes, caches every produced row's abs-sums (and each
// consumer's |Int f - p_k| sum) in FlowSmem::fc and writes the endpoint rows
// seed + h (f + h/2 f') to HBM; every later replay and the endpoint itself
// (MODE_REPLAY_FAST, MODE_ENDPOINT) are scalar-only: the warp-uniform interval
// chains on the cached sums, no coefficient pass, no shuffle reduction.  The
// cached values are the ones the full pass would recompute, bit for bit.
enum : int { MODE_PICARD = 0, MODE_REPLAY = 1, MODE_REPLAY_FAST = 2, MODE_ENDPOINT = 3 };

// Slot indices of the field programs (ct_capi.cu builds them; the quadrotor's
// scalar-only replay below is compiled from the same list).
__host__ __device__ constexpr unsigned char P_(int i) { return static_cast<unsigned char>(i); }
__host__ __device__ constexpr unsigned char T_(int i) { return static_cast<unsigned char>(SLOT_T + i); }
__host__ __device__ constexpr unsigned char V_(int i) { return static_cast<unsigned char>(SLOT_V + i); }
__host__ __device__ constexpr unsigned char C_(int i) { return static_cast<unsigned char>(SLOT_C + i); }

// quadrotor_ode (systems.hpp:24-64) as a field program, U0..U3 the input
// rows (the augmented P12..15 of cl_reach or the held constants C0..3 of
// ct_reach).  X(code, dst, a, b) per entry; constants: kc[0] = 1/mass,
// kc[1] = g, kc[2..7] the inertia ratios.  Each dx_i is consumed once neither
// P_i nor a view of it is read again, so the consumer may overwrite P_i
// (poly_picard's in-place update); independent products run in pairs
// (OP_MUL2 + the OP_MUL after it), the expression trees unchanged.
#define RB_CT_QUAD_OPS(X, U0, U1, U2, U3)                                                       \
  X(OP_CONS, 0, P_(3), 0) X(OP_CONS, 1, P_(4), 0) X(OP_CONS, 2, P_(5), 0) /* dx0..2 = v */     \
  X(OP_SIN, V_(0), P_(6), 0) X(OP_COS, V_(1), P_(6), 0)                   /* sphi, cphi */     \
  X(OP_SIN, V_(2), P_(7), 0) X(OP_COS, V_(3), P_(7), 0)                   /* sth, cth */       \
  X(OP_SIN, V_(4), P_(8), 0) X(OP_COS, V_(5), P_(8), 0)                   /* spsi, cpsi */     \
  X(OP_SCALE, V_(6), U0, 0)                                               /* a = u0 / mass */  \
  X(OP_MUL2, T_(0), V_(1), V_(2)) X(OP_MUL, T_(1), V_(0), V_(4))         /* cphi*sth, sphi*spsi */ \
  X(OP_MUL2, T_(2), T_(0), V_(5)) X(OP_MUL, T_(3), T_(0), V_(4))         /* cs*cpsi, cs*spsi */ \
  X(OP_ADD, T_(2), T_(2), T_(1))                                          /* b3x */            \
  X(OP_MUL2, T_(1), V_(0), V_(5)) X(OP_MUL, T_(0), V_(1), V_(3))         /* sphi*cpsi, b3z */ \
  X(OP_SUB, T_(3), T_(3), T_(1))                                          /* b3y */            \
  X(OP_MUL2, T_(1), V_(6), T_(2)) X(OP_MUL, T_(2), V_(6), T_(3))         /* dx3, dx4 */       \
  X(OP_CONS, 3, T_(1), 0) X(OP_CONS, 4, T_(2), 0)                                              \
  X(OP_INV, V_(7), V_(3), 0)                                              /* tme_inv(cth) */   \
  X(OP_MUL2, T_(3), V_(6), T_(0)) X(OP_MUL, T_(1), V_(2), V_(7))         /* a*b3z, tth */     \
  X(OP_SUBK, T_(3), 0, 1)                                                 /* - gravity */      \
  X(OP_CONS, 5, T_(3), 0)                                                                      \
  X(OP_MUL2, T_(2), V_(0), T_(1)) X(OP_MUL, T_(3), V_(1), T_(1))         /* sphi*tth, cphi*tth */ \
  X(OP_MUL2, T_(2), T_(2), P_(10)) X(OP_MUL, T_(3), T_(3), P_(11))       /* *q, *r */         \
  X(OP_ADD, T_(2), P_(9), T_(2))                                          /* p + ... */        \
  X(OP_ADD, T_(2), T_(2), T_(3))                                          /* dx6 (held) */     \
  X(OP_MUL2, T_(0), V_(1), P_(10)) X(OP_MUL, T_(1), V_(0), P_(11))       /* cphi*q, sphi*r */ \
  X(OP_SUB, T_(0), T_(0), T_(1))                                          /* dx7 (held) */     \
  X(OP_MUL2, T_(1), V_(0), V_(7)) X(OP_MUL, T_(3), V_(1), V_(7))         /* sphi/cth, cphi/cth */ \
  X(OP_MUL2, T_(1), T_(1), P_(10)) X(OP_MUL, T_(3), T_(3), P_(11))       /* *q, *r */         \
  X(OP_ADD, T_(1), T_(1), T_(3))                                          /* dx8 */            \
  X(OP_CONS, 6, T_(2), 0) X(OP_CONS, 7, T_(0), 0) X(OP_CONS, 8, T_(1), 0) /* views of P6..8 dead */ \
  X(OP_MUL2, T_(0), P_(10), P_(11)) X(OP_MUL, T_(1), P_(9), P_(11))      /* q*r, p*r */       \
  X(OP_MUL, T_(2), P_(9), P_(10))                                         /* p*q */            \
  X(OP_SCALE, V_(8), T_(0), 2) X(OP_SCALE, V_(9), U1, 3) X(OP_ADD, T_(0), V_(8), V_(9)) /* dx9 */  \
  X(OP_SCALE, V_(8), T_(1), 4) X(OP_SCALE, V_(9), U2, 5) X(OP_ADD, T_(1), V_(8), V_(9)) /* dx10 */ \
  X(OP_SCALE, V_(8), T_(2), 6) X(OP_SCALE, V_(9), U3, 7) X(OP_ADD, T_(2), V_(8), V_(9)) /* dx11 */ \
  X(OP_CONS, 9, T_(0), 0) X(OP_CONS, 10, T_(1), 0) X(OP_CONS, 11, T_(2), 0)

// Remainder of operator* (taylor_model.hpp:337-359): the excess terms bounded
// over the domain and the remainder interactions, from the operands' scalars.
__device__ __forceinline__ Iv mul_rem(double uc, double vc, double uat, double vat, double au, double av, double bu,
                                      double bv, Iv ur, Iv vr, double h) {
  double sym = au * av;
  sym += (au * bv + av * bu) * h;
  sym += bu * bv * h * h;
  sym += (fabs(uat) * bv + fabs(vat) * bu) * h * h;
  Iv rem{-sym, sym};
  const double tt = uat * vat;
  rem = iadd(rem, imul_0h(h * h, tt));
  const Iv pu = poly_range(uc, au, uat, bu, h), pv = poly_range(vc, av, vat, bv, h);
  rem = iadd(rem, imul(pu, vr));
  rem = iadd(rem, imul(pv, ur));
  return iadd(rem, imul(ur, vr));
}

// operator* (taylor_model.hpp:325-360).  r may alias u or v.
__device__ __forceinline__ void op_mul(double* coef, Slot& r, const Slot& u, const Slot& v, const Lane& L) {
  const double uc = u.c, vc = v.c, uat = u.at, vat = v.at;
  const double au = u.sz, av = v.sz, bu = u.sb, bv = v.sb;
  const Iv ur{u.rlo, u.rhi}, vr{v.rlo, v.rhi};
  const Opnd U = opnd(coef, u), V = opnd(coef, v);
  double* raz = coef + r.az;
  double* rbz = coef + r.bz;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    double ua, ub, va, vb;
    fetch(U, j, ua, ub);
    fetch(V, j, va, vb);
    const double ra = uc * va + vc * ua;
    const double rb = uc * vb + vc * ub + uat * va + vat * ua;
    raz[j] = ra;
    rbz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  const Iv rem = mul_rem(uc, vc, uat, vat, au, av, bu, bv, ur, vr, L.h);
  set_scalars(r, uc * vc, uc * vat + vc * uat, rem, s1, s2);
}

// Two independent products r = u * v, q = x * y in one interleaved pass (ILP
// for the latency-bound warp; each product's arithmetic is op_mul's).  Every
// operand slot is loaded before either result is stored, so q may alias u / v
// and r may alias x / y; r != q, and x, y must not be r.
__device__ __forceinline__ void op_mul2(double* coef, Slot& r, const Slot& u, const Slot& v, Slot& q, const Slot& x,
                                        const Slot& y, const Lane& L) {
  const double uc = u.c, vc = v.c, uat = u.at, vat = v.at, au = u.sz, av = v.sz, bu = u.sb, bv = v.sb;
  const double xc = x.c, yc = y.c, xat = x.at, yat = y.at, ax = x.sz, ay = y.sz, bx = x.sb, by = y.sb;
  const Iv ur{u.rlo, u.rhi}, vr{v.rlo, v.rhi}, xr{x.rlo, x.rhi}, yr{y.rlo, y.rhi};
  const Opnd U = opnd(coef, u), V = opnd(coef, v), X = opnd(coef, x), Y = opnd(coef, y);
  double* raz = coef + r.az;
  double* rbz = coef + r.bz;
  double* qaz = coef + q.az;
  double* qbz = coef + q.bz;
  double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    double ua, ub, va, vb, xa, xb, ya, yb;
    fetch(U, j, ua, ub);
    fetch(V, j, va, vb);
    fetch(X, j, xa, xb);
    fetch(Y, j, ya, yb);
    const double ra = uc * va + vc * ua;
    const double rb = uc * vb + vc * ub + uat * va + vat * ua;
    const double qa = xc * ya + yc * xa;
    const double qb = xc * yb + yc * xb + xat * ya + yat * xa;
    raz[j] = ra;
    rbz[j] = rb;
    qaz[j] = qa;
    qbz[j] = qb;
    s1 += fabs(ra);
    s2 += fabs(rb);
    s3 += fabs(qa);
    s4 += fabs(qb);
  }
  wsum4(s1, s2, s3, s4);
  const Iv rr = mul_rem(uc, vc, uat, vat, au, av, bu, bv, ur, vr, L.h);
  const Iv qr = mul_rem(xc, yc, xat, yat, ax, ay, bx, by, xr, yr, L.h);
  set_scalars(r, uc * vc, uc * vat + vc * uat, rr, s1, s2);
  set_scalars(q, xc * yc, xc * yat + yc * xat, qr, s3, s4);
}

// a + b / a - b (taylor_model.hpp:245-269); r may alias a or b.
__device__ __forceinline__ void op_addsub(double* coef, Slot& r, const Slot& a, const Slot& b, bool sub,
                                          const Lane& L) {
  const double c = sub ? a.c - b.c : a.c + b.c;
  const double at = sub ? a.at - b.at : a.at + b.at;
  const Iv rem = sub ? isub(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi}) : iadd(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi});
  const Opnd A = opnd(coef, a), B = opnd(coef, b);
  double* raz = coef + r.az;
  double* rbz = coef + r.bz;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    double aa, ab, ba, bb;
    fetch(A, j, aa, ab);
    fetch(B, j, ba, bb);
    const double ra = sub ? aa - ba : aa + ba;
    const double rb = sub ? ab - bb : ab + bb;
    raz[j] = ra;
    rbz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  set_scalars(r, c, at, rem, s1, s2);
}

// r = a, a view materialized into a stored row (no reference counterpart: the
// reference's views are ordinary TMExpr values).
__device__ __noinline__ void op_copy(double* coef, Slot& r, const Slot& a, const Lane L) {
  const Opnd A = opnd(coef, a);
  double* raz = coef + r.az;
  double* rbz = coef + r.bz;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    double aa, ab;
    fetch(A, j, aa, ab);
    raz[j] = aa;
    rbz[j] = ab;
    s1 += fabs(aa);
    s2 += fabs(ab);
  }
  wsum2(s1, s2);
  set_scalars(r, a.c, a.at, Iv{a.rlo, a.rhi}, s1, s2);
}

// r = view of u scaled by s: r.az = (u.az * s) (taylor_model.hpp:284-295).
__device__ __forceinline__ void make_view(Slot& r, const Slot& u, double s) {
  r.az = u.az;
  r.bz = u.bz;
  r.view = 1;
  if (u.view) {
    r.s1 = u.s1;
    r.s2 = s;
  } else {
    r.s1 = s;
    r.s2 = 1.0;
  }
}

// Scalar-only forms of the stored-row operations for the fast replays: the
// result's scalars from its operands' scalars, its abs-sums from the cache.
// Every operand scalar is read before the result is written (r may alias).
__device__ __forceinline__ void mul_fast(Slot& r, const Slot& u, const Slot& v, double2 sums, double h) {
  const double uc = u.c, vc = v.c, uat = u.at, vat = v.at;
  const Iv rem = mul_rem(uc, vc, uat, vat, u.sz, v.sz, u.sb, v.sb, Iv{u.rlo, u.rhi}, Iv{v.rlo, v.rhi}, h);
  set_scalars(r, uc * vc, uc * vat + vc * uat, rem, sums.x, sums.y);
}
__device__ __forceinline__ void mul2_fast(Slot& r, const Slot& u, const Slot& v, double2 rs, Slot& q, const Slot& x,
                                          const Slot& y, double2 qs, double h) {
  const double uc = u.c, vc = v.c, uat = u.at, vat = v.at, xc = x.c, yc = y.c, xat = x.at, yat = y.at;
  const Iv rr = mul_rem(uc, vc, uat, vat, u.sz, v.sz, u.sb, v.sb, Iv{u.rlo, u.rhi}, Iv{v.rlo, v.rhi}, h);
  const Iv qr = mul_rem(xc, yc, xat, yat, x.sz, y.sz, x.sb, y.sb, Iv{x.rlo, x.rhi}, Iv{y.rlo, y.rhi}, h);
  set_scalars(r, uc * vc, uc * vat + vc * uat, rr, rs.x, rs.y);
  set_scalars(q, xc * yc, xc * yat + yc * xat, qr, qs.x, qs.y);
}
__device__ __forceinline__ void addsub_fast(Slot& r, const Slot& a, const Slot& b, bool sub, double2 sums) {
  const double c = sub ? a.c - b.c : a.c + b.c;
  const double at = sub ? a.at - b.at : a.at + b.at;
  const Iv rem = sub ? isub(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi}) : iadd(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi});
  set_scalars(r, c, at, rem, sums.x, sums.y);
}

// The field program on the slots; `mode` selects what CONS does with dx_i:
//   PICARD        g_i = seed_i + Int dx_i written over P_i (flowpipe_ct.hpp:130-133)
//   REPLAY(_FAST) I1_i = range(seed_i + Int dx_i - p_k,i) (:154-165); the full
//                 replay also writes x(h)_i's rows seed_i + h (dx_i + h/2 dx_i')
//                 to the state's HBM rows (:241-257)
//   ENDPOINT      x(h)_i's centre and remainder (scalar-only)
// Returns the tme_inv "throw" (taylor_model.hpp:367-368).
__device__ __noinline__ bool run_field(FlowSmem& W, int prog, int mode, const Lane L, double* gM) {
  bool thrown = false;
  const double h = L.h;
  const int lane = L.lane;
  const bool fast = mode >= MODE_REPLAY_FAST, record = mode == MODE_REPLAY;
  double* coef = flow_coef<false>(W);
  double2* fc = W.fc_s;  // indexed by pc - prog
  TOp next = kProgs[prog];
  for (int pc = prog;; ++pc) {
    const TOp op = next;
    if (op.code == OP_END) break;
    next = kProgs[pc + 1];  // dispatch of the next op overlaps this one
    switch (op.code) {
      case OP_MUL: {
        Slot& r = W.D[op.dst];
        if (fast) {
          mul_fast(r, W.D[op.a], W.D[op.b], fc[pc - prog], h);
        } else {
          op_mul(coef, r, W.D[op.a], W.D[op.b], L);
          if (record && lane == 0) fc[pc - prog] = make_double2(r.sz, r.sb);
        }
        break;
      }
      case OP_MUL2: {  // this entry and the next one (an OP_MUL) as one pass
        const TOp o2 = next;
        ++pc;
        next = kProgs[pc + 1];
        Slot& r = W.D[op.dst];
        Slot& q = W.D[o2.dst];
        if (fast) {
          mul2_fast(r, W.D[op.a], W.D[op.b], fc[pc - 1 - prog], q, W.D[o2.a], W.D[o2.b], fc[pc - prog], h);
        } else {
          op_mul2(coef, r, W.D[op.a], W.D[op.b], q, W.D[o2.a], W.D[o2.b], L);
          if (record && lane == 0) {
            fc[pc - 1 - prog] = make_double2(r.sz, r.sb);
            fc[pc - prog] = make_double2(q.sz, q.sb);
          }
        }
        break;
      }
      case OP_ADD:
      case OP_SUB: {
        Slot& r = W.D[op.dst];
        if (fast) {
          addsub_fast(r, W.D[op.a], W.D[op.b], op.code == OP_SUB, fc[pc - prog]);
        } else {
          op_addsub(coef, r, W.D[op.a], W.D[op.b], op.code == OP_SUB, L);
          if (record && lane == 0) fc[pc - prog] = make_double2(r.sz, r.sb);
        }
        break;
      }
      case OP_COPY: {
        Slot& r = W.D[op.dst];
        if (fast) {
          const Slot& a = W.D[op.a];
          set_scalars(r, a.c, a.at, Iv{a.rlo, a.rhi}, fc[pc - prog].x, fc[pc - prog].y);
        } else {
          op_copy(coef, r, W.D[op.a], L);
          if (record && lane == 0) fc[pc - prog] = make_double2(r.sz, r.sb);
        }
        break;
      }
      case OP_SUBK:
        W.D[op.dst].c = W.D[op.dst].c - W.kc[op.b];
        break;
      case OP_CONST: {  // tme_const (taylor_model.hpp:240-243)
        Slot& r = W.D[op.dst];
        set_scalars(r, W.kc[op.b], 0.0, Iv{0.0, 0.0}, 0.0, 0.0);
        r.az = W.off_zero;
        r.bz = W.off_zero;
        r.view = 0;
        r.s1 = r.s2 = 1.0;
        break;
      }
      case OP_SCALE: {  // TM * s (taylor_model.hpp:297-300)
        const Slot& u = W.D[op.a];
        Slot& r = W.D[op.dst];
        const double s = W.kc[op.b];
        const Iv rem = iscale(s, Iv{u.rlo, u.rhi});
        set_scalars(r, u.c * s, u.at * s, rem, fabs(s) * u.sz, fabs(s) * u.sb);
        make_view(r, u, s);
        break;
      }
      case OP_SIN:
      case OP_COS: {  // linearization about the centre (taylor_model.hpp:397-425)
        const Slot& u = W.D[op.a];
        Slot& r = W.D[op.dst];
        const double m = u.c;
        const Iv range = iadd(poly_range(u.c, u.sz, u.at, u.sb, h), Iv{u.rlo, u.rhi});
        const double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
        const double err = rad * rad * 0.5;
        double sm, cm;
        sincos(m, &sm, &cm);
        const bool isc = op.code == OP_COS;
        const double s = isc ? -sm : cm;
        Iv rem = iscale(s, Iv{u.rlo, u.rhi});
        rem = iadd(rem, Iv{-err, err});
        set_scalars(r, (m - m) * s + (isc ? cm : sm), u.at * s, rem, fabs(s) * u.sz, fabs(s) * u.sb);
        make_view(r, u, s);
        break;
      }
      case OP_INV: {  // tme_inv (taylor_model.hpp:364-380)
        const Slot& v = W.D[op.a];
        Slot& r = W.D[op.dst];
        const Iv range = iadd(poly_range(v.c, v.sz, v.at, v.sb, h), Iv{v.rlo, v.rhi});
        if (range.lo <= 0.0 && range.hi >= 0.0) thrown = true;
        const double m = v.c, mm = m * m;
        const double e_lo = 1.0 / range.lo - (2.0 / m - range.lo / mm);
        const double e_hi = 1.0 / range.hi - (2.0 / m - range.hi / mm);
        const Iv e{smin(smin(e_lo, e_hi), 0.0), smax(smax(e_lo, e_hi), 0.0)};
        const double s = -1.0 / mm;
        Iv rem = iscale(s, Iv{v.rlo, v.rhi});
        rem = iadd(rem, e);
        set_scalars(r, v.c * s + 2.0 / m, v.at * s, rem, fabs(s) * v.sz, fabs(s) * v.sb);
        make_view(r, v, s);
        break;
      }
      case OP_CONS:
      case OP_CONS0: {
        const int i = op.dst;
        const bool zero = op.code == OP_CONS0;
        const Slot& f = W.D[zero ? 0 : op.a];
        const Opnd F = opnd(coef, f);
        const double fc_ = zero ? 0.0 : f.c, fat = zero ? 0.0 : f.at;
        const double fsz = zero ? 0.0 : f.sz, fsb = zero ? 0.0 : f.sb;
        const Iv fr = zero ? Iv{0.0, 0.0} : Iv{f.rlo, f.rhi};
        const double* S = coef + i * NZP;
        double* Pb = coef + W.pbz[i];
        if (mode == MODE_ENDPOINT) {  // the rows were written by this step's full replay
          W.ec[i] = W.sc[i] + h * (fc_ + fat * h * 0.5);
          W.erem_s[i] = iadd(imul(Iv{h, h}, fr), Iv{0.0, 0.0});
          break;
        }
        // tme_integrate(dx_i) remainder (taylor_model.hpp:436-443)
        const double half_at = fat * 0.5;
        Iv rem = imul_0h(h * h, half_at);
        const double bb = fsb * h * h * 0.5;
        rem = iadd(rem, Iv{-bb, bb});
        rem = iadd(rem, imul(fr, Iv{0.0, h}));
        if (mode == MODE_PICARD) {
          if (W.own[i]) {  // aliased rows: bz is S_j or 0 by construction
#pragma unroll
            for (int k = 0; k < NZC; ++k) {
              if (!L.act[k]) continue;
              const int j = lane + 32 * k;
              double fa = 0.0, fb;
              if (!zero) fetch(F, j, fa, fb);
              Pb[j] = fa;
            }
          }
          set_scalars(W.D[i], W.sc[i], fc_, rem, W.ssz[i], fsz);
        } else {  // REPLAY: (seed + Int f) - p_k; its z part seed - p_k.az is exactly 0
          double s2;
          if (fast) {
            s2 = fc[pc - prog].x;
          } else {
            s2 = 0.0;
#pragma unroll
            for (int k = 0; k < NZC; ++k) {
              if (!L.act[k]) continue;
              const int j = lane + 32 * k;
              double fa = 0.0, fb = 0.0;
              if (!zero) fetch(F, j, fa, fb);
              s2 += fabs(fa - Pb[j]);
              gM[i * NZP + j] = S[j] + h * (fa + fb * h * 0.5);  // the endpoint row (:241-257)
            }
            s2 = wsum(s2);
            if (lane == 0) fc[pc - prog] = make_double2(s2, 0.0);
          }
          const Slot& pk = W.D[i];
          const double zr = isfinite(W.ssz[i]) ? 0.0 : W.ssz[i] - W.ssz[i];
          W.nx_s[i] = iadd(poly_range(W.sc[i] - pk.c, zr, fc_ - pk.at, s2, h), rem);
        }
        break;
      }
      default:
        break;
    }
  }
  return thrown;
}

// The quadrotor program's scalar-only replay / endpoint (MODE_REPLAY_FAST,
// MODE_ENDPOINT) compiled from RB_CT_QUAD_OPS instead of interpreted: the slot
// scalars live in registers (compile-time slot indices) and the compiler
// schedules the program's independent chains side by side (sin / cos of the
// three angles, the two product trees, dx9..11) instead of one interpreted
// operation after another.  Each operation is run_field's fast form, operand
// order included; the abs-sums come from this step's full replay (FlowSmem::fc).
// The quadrotor programs' row layout as compile-time constants (what the
// flow kernel derives from CTParams::bzsrc; the host selects the compiled
// programs only when the two agree, ct_capi.cu): rows 0..2 integrate
// P3..5 (bz = S3..5), rows 3..11 own their Picard bz rows, the input rows
// 12..15 of the augmented field have udot = 0 (bz = the zero row).  Constant
// row offsets let the compiler prove which shared-memory rows an operation
// touches and move the next operations' loads ahead of this one's stores.
template <bool HELD, bool CMP = false>
struct QuadLayout {
  static constexpr int rs = CMP ? kRowC : NZP;  // row stride
  static constexpr int na = HELD ? NX : NA;
  static constexpr int off_zero = CMP ? kNoRow : na * rs;
  static constexpr int off_pbz = na * rs + (CMP ? 0 : rs);
  static constexpr int npb = 9;
  static constexpr int off_taz = off_pbz + npb * rs;
  static constexpr int off_tbz = off_taz + NTF * rs;
  __host__ __device__ static constexpr int pbz(int i) {
    return i < 3 ? (i + 3) * rs : i < 12 ? off_pbz + (i - 3) * rs : off_zero;
  }
  __host__ __device__ static constexpr bool own(int i) { return i >= 3 && i < 12; }
};
// a coefficient of row `row` (kNoRow: the zero row, absent in the compact layout)
__device__ __forceinline__ double rowv(const double* coef, int row, int j) { return row < 0 ? 0.0 : coef[row + j]; }

struct FS {
  double c, at, rlo, rhi, sz, sb;
};
// Between two replays of a step only the remainders change, so everything
// else each operation computes is recorded by the step's first scalar-only
// replay (CACHED = false) into the temporaries' coefficient rows (dead until
// the next step's Picard iteration; kFastK doubles per program entry), and
// the later replays and the endpoint (CACHED = true) carry the remainders
// only: operator* as base + pu * vr + pv * ur + ur * vr with base = the excess
// interval + the tau^2 term and pu / pv the operands' polynomial ranges
// (taylor_model.hpp:337-359, the same additions in the same order);
// sin / cos / reciprocal from the cached range without the remainder and the
// linearization point; the consumers from their cached constant parts.
constexpr int kFastK = 6;
template <int CODE, int DST, int A, int B, bool CACHED>
__device__ __forceinline__ void fast_op(FS (&D)[NSLOT], FlowSmem& W, const Side& X, double* K, int pc, int mode,
                                        double h, bool& thrown, bool rec) {
  double* k = K + pc * kFastK;
  if constexpr (CODE == OP_MUL || CODE == OP_MUL2) {  // the pair's second entry follows as an OP_MUL
    const FS u = D[A], v = D[B];
    const Iv ur{u.rlo, u.rhi}, vr{v.rlo, v.rhi};
    Iv base, pu, pv;
    if constexpr (CACHED) {
      base = Iv{k[0], k[1]};
      pu = Iv{k[2], k[3]};
      pv = Iv{k[4], k[5]};
    } else {  // mul_rem's constant part
      const double uc = u.c, vc = v.c, uat = u.at, vat = v.at, au = u.sz, av = v.sz, bu = u.sb, bv = v.sb;
      double sym = au * av;
      sym += (au * bv + av * bu) * h;
      sym += bu * bv * h * h;
      sym += (fabs(uat) * bv + fabs(vat) * bu) * h * h;
      base = iadd(Iv{-sym, sym}, imul_0h(h * h, uat * vat));
      pu = poly_range(uc, au, uat, bu, h);
      pv = poly_range(vc, av, vat, bv, h);
      if (rec) {
        k[0] = base.lo; k[1] = base.hi; k[2] = pu.lo; k[3] = pu.hi; k[4] = pv.lo; k[5] = pv.hi;
      }
    }
    Iv rem = iadd(base, imul(pu, vr));
    rem = iadd(rem, imul(pv, ur));
    rem = iadd(rem, imul(ur, vr));
    if constexpr (CACHED) {
      D[DST].rlo = rem.lo;
      D[DST].rhi = rem.hi;
    } else {
      const double2 s = X.fc[pc];
      D[DST] = FS{u.c * v.c, u.c * v.at + v.c * u.at, rem.lo, rem.hi, s.x, s.y};
    }
  } else if constexpr (CODE == OP_ADD || CODE == OP_SUB) {
    const FS a = D[A], b = D[B];
    constexpr bool sub = CODE == OP_SUB;
    const Iv rem = sub ? isub(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi}) : iadd(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi});
    if constexpr (CACHED) {
      D[DST].rlo = rem.lo;
      D[DST].rhi = rem.hi;
    } else {
      const double2 s = X.fc[pc];
      D[DST] = FS{sub ? a.c - b.c : a.c + b.c, sub ? a.at - b.at : a.at + b.at, rem.lo, rem.hi, s.x, s.y};
    }
  } else if constexpr (CODE == OP_SUBK) {
    if constexpr (!CACHED) D[DST].c = D[DST].c - W.kc[B];
  } else if constexpr (CODE == OP_CONST) {
    D[DST] = FS{W.kc[B], 0.0, 0.0, 0.0, 0.0, 0.0};
  } else if constexpr (CODE == OP_SCALE) {
    const FS u = D[A];
    const double s = W.kc[B];
    const Iv rem = iscale(s, Iv{u.rlo, u.rhi});
    if constexpr (CACHED) {
      D[DST].rlo = rem.lo;
      D[DST].rhi = rem.hi;
    } else {
      D[DST] = FS{u.c * s, u.at * s, rem.lo, rem.hi, fabs(s) * u.sz, fabs(s) * u.sb};
    }
  } else if constexpr (CODE == OP_SIN || CODE == OP_COS) {
    const FS u = D[A];
    Iv pr;
    double m, s;
    double sm = 0.0, cm = 0.0;
    constexpr bool isc = CODE == OP_COS;
    if constexpr (CACHED) {
      pr = Iv{k[0], k[1]};
      m = k[2];
      s = k[3];
    } else {
      m = u.c;
      pr = poly_range(u.c, u.sz, u.at, u.sb, h);
      sincos(m, &sm, &cm);
      s = isc ? -sm : cm;
      if (rec) {
        k[0] = pr.lo; k[1] = pr.hi; k[2] = m; k[3] = s;
      }
    }
    const Iv range = iadd(pr, Iv{u.rlo, u.rhi});
    const double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
    const double err = rad * rad * 0.5;
    Iv rem = iscale(s, Iv{u.rlo, u.rhi});
    rem = iadd(rem, Iv{-err, err});
    if constexpr (CACHED) {
      D[DST].rlo = rem.lo;
      D[DST].rhi = rem.hi;
    } else {
      D[DST] = FS{(m - m) * s + (isc ? cm : sm), u.at * s, rem.lo, rem.hi, fabs(s) * u.sz, fabs(s) * u.sb};
    }
  } else if constexpr (CODE == OP_INV) {
    const FS v = D[A];
    Iv pr;
    double m, mm;
    if constexpr (CACHED) {
      pr = Iv{k[0], k[1]};
      m = k[2];
      mm = k[3];
    } else {
      pr = poly_range(v.c, v.sz, v.at, v.sb, h);
      m = v.c;
      mm = m * m;
      if (rec) {
        k[0] = pr.lo; k[1] = pr.hi; k[2] = m; k[3] = mm;
      }
    }
    const Iv range = iadd(pr, Iv{v.rlo, v.rhi});
    if (range.lo <= 0.0 && range.hi >= 0.0) thrown = true;
    const double e_lo = 1.0 / range.lo - (2.0 / m - range.lo / mm);
    const double e_hi = 1.0 / range.hi - (2.0 / m - range.hi / mm);
    const Iv e{smin(smin(e_lo, e_hi), 0.0), smax(smax(e_lo, e_hi), 0.0)};
    const double s = -1.0 / mm;
    Iv rem = iscale(s, Iv{v.rlo, v.rhi});
    rem = iadd(rem, e);
    if constexpr (CACHED) {
      D[DST].rlo = rem.lo;
      D[DST].rhi = rem.hi;
    } else {
      D[DST] = FS{v.c * s + 2.0 / m, v.at * s, rem.lo, rem.hi, fabs(s) * v.sz, fabs(s) * v.sb};
    }
  } else if constexpr (CODE == OP_CONS || CODE == OP_CONS0) {
    constexpr int i = DST;
    constexpr bool zero = CODE == OP_CONS0;
    const FS f = D[zero ? 0 : A];
    const Iv fr = zero ? Iv{0.0, 0.0} : Iv{f.rlo, f.rhi};
    Iv ca, cb;  // tme_integrate's constant part, the polynomial range of (seed + Int f) - p_k
    double ec;
    if constexpr (CACHED) {
      ca = Iv{k[0], k[1]};
      cb = Iv{k[2], k[3]};
      ec = k[4];
    } else {
      const double fc_ = zero ? 0.0 : f.c, fat = zero ? 0.0 : f.at, fsb = zero ? 0.0 : f.sb;
      ec = W.sc[i] + h * (fc_ + fat * h * 0.5);
      const double half_at = fat * 0.5;
      const double bb = fsb * h * h * 0.5;
      ca = iadd(imul_0h(h * h, half_at), Iv{-bb, bb});
      const FS pk = D[i];
      const double zr = isfinite(W.ssz[i]) ? 0.0 : W.ssz[i] - W.ssz[i];
      cb = poly_range(W.sc[i] - pk.c, zr, fc_ - pk.at, X.fc[pc].x, h);
      if (rec) {
        k[0] = ca.lo; k[1] = ca.hi; k[2] = cb.lo; k[3] = cb.hi; k[4] = ec;
      }
    }
    if (mode == MODE_ENDPOINT) {
      W.ec[i] = ec;
      X.erem[i] = iadd(imul(Iv{h, h}, fr), Iv{0.0, 0.0});
    } else {
      const Iv rem = iadd(ca, imul(fr, Iv{0.0, h}));
      X.nx[i] = iadd(cb, rem);
    }
  }
}

// HELD: ct_reach's quadrotor field (inputs C0..3 from kc[8..11], four OP_CONST
// entries first); else cl_reach's augmented field (inputs P12..15, udot = 0).
// CACHED = false with rec: record the constants (lane 0) for the CACHED calls.
template <bool HELD, bool CACHED, bool CMP = false>
__device__ __noinline__ bool quad_fast(FlowSmem& W, const Side X, int mode, double h, bool rec) {
  FS D[NSLOT];
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const Slot& p = W.D[i];
    D[i] = FS{p.c, p.at, p.rlo, p.rhi, p.sz, p.sb};
  }
  double* K = flow_coef<CMP>(W) + QuadLayout<HELD, CMP>::off_taz;
  rec = rec && (threadIdx.x & 31) == 0;
  bool thrown = false;
  int pc = 0;
#define RB_CT_FAST_OP(c, d, a, b) fast_op<c, d, a, b, CACHED>(D, W, X, K, pc++, mode, h, thrown, rec);
  if constexpr (HELD) {
    RB_CT_FAST_OP(OP_CONST, C_(0), 0, 8)
    RB_CT_FAST_OP(OP_CONST, C_(1), 0, 9)
    RB_CT_FAST_OP(OP_CONST, C_(2), 0, 10)
    RB_CT_FAST_OP(OP_CONST, C_(3), 0, 11)
    RB_CT_QUAD_OPS(RB_CT_FAST_OP, C_(0), C_(1), C_(2), C_(3))
  } else {
    RB_CT_QUAD_OPS(RB_CT_FAST_OP, P_(12), P_(13), P_(14), P_(15))
    RB_CT_FAST_OP(OP_CONS0, 12, 0, 0)
    RB_CT_FAST_OP(OP_CONS0, 13, 0, 0)
    RB_CT_FAST_OP(OP_CONS0, 14, 0, 0)
    RB_CT_FAST_OP(OP_CONS0, 15, 0, 0)
  }
#undef RB_CT_FAST_OP
  return thrown;
}

// The full-mode passes (MODE_PICARD, MODE_REPLAY) of the quadrotor program,
// compiled from RB_CT_QUAD_OPS like quad_fast: slot scalars, view scales and
// row offsets in registers, the coefficient rows in shared memory.  Each
// operation is run_field's (operand order, excess folding, the abs-sum
// butterflies), but with the program known to the compiler one operation's
// scalar chain and shuffle reduction overlap the next operations' coefficient
// passes instead of serializing through the interpreter's dispatch.
struct FR {
  double c, at, rlo, rhi, sz, sb;
  double s;    // view scale (1 for a stored row)
  int az, bz;  // coefficient rows (offsets into FlowSmem::coef())
};
struct FullCtx {
  FlowSmem& W;
  double* coef;
  double* gM;
  const Lane& L;
  int mode;
  Side sd;
};
template <int CODE, int DST, int A, int B, bool HELD, bool CMP>
__device__ __forceinline__ void full_op(FR (&D)[NSLOT], const FullCtx& X, int pc, bool& thrown) {
  using Q = QuadLayout<HELD, CMP>;
  FlowSmem& W = X.W;
  double* coef = X.coef;
  const Lane& L = X.L;
  const double h = L.h;
  const int lane = L.lane;
  const bool record = X.mode == MODE_REPLAY;
  if constexpr (CODE == OP_MUL || CODE == OP_MUL2 || CODE == OP_ADD || CODE == OP_SUB) {
    static_assert(DST >= SLOT_T && DST < SLOT_V, "stored results go to temporaries");
    const FR u = D[A], v = D[B];
    constexpr int raz = Q::off_taz + (DST - SLOT_T) * Q::rs, rbz = Q::off_tbz + (DST - SLOT_T) * Q::rs;
    constexpr bool mul = CODE == OP_MUL || CODE == OP_MUL2, sub = CODE == OP_SUB;
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int k = 0; k < NZC; ++k) {
      if (!L.act[k]) continue;
      const int j = lane + 32 * k;
      // stored rows (P, T, C slots) have scale 1: x * 1.0 == x, so only views multiply
      constexpr bool uv = A >= SLOT_V && A < SLOT_C, vv = B >= SLOT_V && B < SLOT_C;
      const double uaz = rowv(coef, u.az, j), ubz = rowv(coef, u.bz, j);
      const double vaz = rowv(coef, v.az, j), vbz = rowv(coef, v.bz, j);
      const double ua = uv ? uaz * u.s : uaz, ub = uv ? ubz * u.s : ubz;
      const double va = vv ? vaz * v.s : vaz, vb = vv ? vbz * v.s : vbz;
      double ra, rb;
      if constexpr (mul) {
        ra = u.c * va + v.c * ua;
        rb = u.c * vb + v.c * ub + u.at * va + v.at * ua;
      } else {
        ra = sub ? ua - va : ua + va;
        rb = sub ? ub - vb : ub + vb;
      }
      coef[raz + j] = ra;
      coef[rbz + j] = rb;
      s1 += fabs(ra);
      s2 += fabs(rb);
    }
    wsum2(s1, s2);
    FR r;
    if constexpr (mul) {
      const Iv rem = mul_rem(u.c, v.c, u.at, v.at, u.sz, v.sz, u.sb, v.sb, Iv{u.rlo, u.rhi}, Iv{v.rlo, v.rhi}, h);
      r = FR{u.c * v.c, u.c * v.at + v.c * u.at, rem.lo, rem.hi, s1, s2, 1.0, raz, rbz};
    } else {
      const Iv rem = sub ? isub(Iv{u.rlo, u.rhi}, Iv{v.rlo, v.rhi}) : iadd(Iv{u.rlo, u.rhi}, Iv{v.rlo, v.rhi});
      r = FR{sub ? u.c - v.c : u.c + v.c, sub ? u.at - v.at : u.at + v.at, rem.lo, rem.hi, s1, s2, 1.0, raz, rbz};
    }
    D[DST] = r;
    if (record && lane == 0) X.sd.fc[pc] = make_double2(s1, s2);
  } else if constexpr (CODE == OP_SUBK) {
    D[DST].c = D[DST].c - W.kc[B];
  } else if constexpr (CODE == OP_CONST) {
    D[DST] = FR{W.kc[B], 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, Q::off_zero, Q::off_zero};
  } else if constexpr (CODE == OP_SCALE) {
    const FR u = D[A];
    const double s = W.kc[B];
    const Iv rem = iscale(s, Iv{u.rlo, u.rhi});
    D[DST] = FR{u.c * s, u.at * s, rem.lo, rem.hi, fabs(s) * u.sz, fabs(s) * u.sb, u.s * s, u.az, u.bz};
  } else if constexpr (CODE == OP_SIN || CODE == OP_COS) {
    const FR u = D[A];
    const double m = u.c;
    const Iv range = iadd(poly_range(u.c, u.sz, u.at, u.sb, h), Iv{u.rlo, u.rhi});
    const double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
    const double err = rad * rad * 0.5;
    double sm, cm;
    sincos(m, &sm, &cm);
    constexpr bool isc = CODE == OP_COS;
    const double s = isc ? -sm : cm;
    Iv rem = iscale(s, Iv{u.rlo, u.rhi});
    rem = iadd(rem, Iv{-err, err});
    D[DST] = FR{(m - m) * s + (isc ? cm : sm), u.at * s, rem.lo, rem.hi, fabs(s) * u.sz, fabs(s) * u.sb, u.s * s,
                u.az, u.bz};
  } else if constexpr (CODE == OP_INV) {
    const FR v = D[A];
    const Iv range = iadd(poly_range(v.c, v.sz, v.at, v.sb, h), Iv{v.rlo, v.rhi});
    if (range.lo <= 0.0 && range.hi >= 0.0) thrown = true;
    const double m = v.c, mm = m * m;
    const double e_lo = 1.0 / range.lo - (2.0 / m - range.lo / mm);
    const double e_hi = 1.0 / range.hi - (2.0 / m - range.hi / mm);
    const Iv e{smin(smin(e_lo, e_hi), 0.0), smax(smax(e_lo, e_hi), 0.0)};
    const double s = -1.0 / mm;
    Iv rem = iscale(s, Iv{v.rlo, v.rhi});
    rem = iadd(rem, e);
    D[DST] = FR{v.c * s + 2.0 / m, v.at * s, rem.lo, rem.hi, fabs(s) * v.sz, fabs(s) * v.sb, v.s * s, v.az, v.bz};
  } else if constexpr (CODE == OP_CONS || CODE == OP_CONS0) {
    constexpr int i = DST;
    constexpr bool zero = CODE == OP_CONS0;
    const FR f = D[zero ? 0 : A];
    const double fc_ = zero ? 0.0 : f.c, fat = zero ? 0.0 : f.at, fsz = zero ? 0.0 : f.sz, fsb = zero ? 0.0 : f.sb;
    const Iv fr = zero ? Iv{0.0, 0.0} : Iv{f.rlo, f.rhi};
    const double* S = coef + i * Q::rs;
    double* Pb = coef + (Q::pbz(i) < 0 ? 0 : Q::pbz(i));
    const double half_at = fat * 0.5;
    Iv rem = imul_0h(h * h, half_at);
    const double bb = fsb * h * h * 0.5;
    rem = iadd(rem, Iv{-bb, bb});
    rem = iadd(rem, imul(fr, Iv{0.0, h}));
    if (X.mode == MODE_PICARD) {
      if constexpr (Q::own(i)) {
#pragma unroll
        for (int k = 0; k < NZC; ++k) {
          if (!L.act[k]) continue;
          const int j = lane + 32 * k;
          Pb[j] = zero ? 0.0 : rowv(coef, f.az, j) * f.s;
        }
      }
      set_scalars(W.D[i], W.sc[i], fc_, rem, W.ssz[i], fsz);
    } else {  // the step's full replay: range of (seed + Int f) - p_k, the endpoint rows, the cached sum
      double s2 = 0.0;
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        if (!L.act[k]) continue;
        const int j = lane + 32 * k;
        const double fa = zero ? 0.0 : rowv(coef, f.az, j) * f.s, fb = zero ? 0.0 : rowv(coef, f.bz, j) * f.s;
        s2 += fabs(fa - (Q::pbz(i) < 0 ? 0.0 : Pb[j]));
        X.gM[i * NZP + j] = S[j] + h * (fa + fb * h * 0.5);
      }
      s2 = wsum(s2);
      if (lane == 0) X.sd.fc[pc] = make_double2(s2, 0.0);
      const FR pk = D[i];
      const double zr = isfinite(W.ssz[i]) ? 0.0 : W.ssz[i] - W.ssz[i];
      X.sd.nx[i] = iadd(poly_range(W.sc[i] - pk.c, zr, fc_ - pk.at, s2, h), rem);
    }
  }
}

template <bool HELD, bool CMP = false>
__device__ __noinline__ bool quad_full(FlowSmem& W, const Side sd, int mode, const Lane L, double* gM) {
  using Q = QuadLayout<HELD, CMP>;
  FR D[NSLOT];
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    const Slot& p = W.D[i];
    D[i] = FR{p.c, p.at, p.rlo, p.rhi, p.sz, p.sb, 1.0, i * Q::rs, Q::pbz(i)};
  }
  const FullCtx X{W, flow_coef<CMP>(W), gM, L, mode, sd};
  bool thrown = false;
  int pc = 0;
#define RB_CT_FULL_OP(c, d, a, b) full_op<c, d, a, b, HELD, CMP>(D, X, pc++, thrown);
  if constexpr (HELD) {
    RB_CT_FULL_OP(OP_CONST, C_(0), 0, 8)
    RB_CT_FULL_OP(OP_CONST, C_(1), 0, 9)
    RB_CT_FULL_OP(OP_CONST, C_(2), 0, 10)
    RB_CT_FULL_OP(OP_CONST, C_(3), 0, 11)
    RB_CT_QUAD_OPS(RB_CT_FULL_OP, C_(0), C_(1), C_(2), C_(3))
  } else {
    RB_CT_QUAD_OPS(RB_CT_FULL_OP, P_(12), P_(13), P_(14), P_(15))
    RB_CT_FULL_OP(OP_CONS0, 12, 0, 0)
    RB_CT_FULL_OP(OP_CONS0, 13, 0, 0)
    RB_CT_FULL_OP(OP_CONS0, 14, 0, 0)
    RB_CT_FULL_OP(OP_CONS0, 15, 0, 0)
  }
#undef RB_CT_FULL_OP
  return thrown;
}

__device__ __forceinline__ void emit_box(const CTParams& P, long long b, int k, int na, int d, double lo, double hi) {
  if (!P.split) {
    const size_t o = (static_cast<size_t>(b) * P.T + k) * na + d;
    P.out_lo[o] = lo;
    P.out_hi[o] = hi;
  } else {
    if (lo == lo) atomicMin(&P.hull_lo[k * na + d], order_key(lo));
    if (hi == hi) atomicMax(&P.hull_hi[k * na + d], order_key(hi));
    if (P.part_begin + b == 0) {
      if (lo != lo) P.hull_nan0[(k * na + d) * 2 + 0] = 1;
      if (hi != hi) P.hull_nan0[(k * na + d) * 2 + 1] = 1;
    }
    if (!(isfinite(lo) && isfinite(hi))) atomicOr(&P.hull_div[k], 1);
  }
}

// Per-sample outputs at the end of the run (tube mode) or the hull's
// min box count / failure key (split mode, refine.hpp:133-148).
__device__ __forceinline__ void finalize(const CTParams& P, long long b, int nb, int st, int fs) {
  if (!P.split) {
    P.n_boxes[b] = nb;
    P.failed_step[b] = fs;
    P.status[b] = st;
  } else {
    atomicMin(P.hull_nboxes, nb);
    if (st != CT_OK) {
      const unsigned long long key = (static_cast<unsigned long long>(fs >= 0 ? fs : nb) << 40) |
                                     (static_cast<unsigned long long>(P.part_begin + b) << 8) |
                                     static_cast<unsigned long long>(st & 0xff);
      atomicMin(P.hull_fail_key, key);
    }
  }
}

// Initial box of sample b, dimension d: a batch row, or part b of split_box
// (refine.hpp:83-115, last dimension fastest).
__device__ __forceinline__ void x0_box(const CTParams& P, long long b, int d, double& lo, double& hi) {
  if (P.split) {
    long long p = P.part_begin + b;
    for (int e = P.n - 1; e >= 0; --e) {
      const int k = P.counts[e];
      const int i = static_cast<int>(p % k);
      p /= k;
      if (e == d) {
        const double xl = P.sx_lo[e], xh = P.sx_hi[e];
        lo = (i == 0) ? xl : xl + (xh - xl) * (static_cast<double>(i) / k);
        hi = (i + 1 == k) ? xh : xl + (xh - xl) * (static_cast<double>(i + 1) / k);
      }
    }
  } else {
    lo = P.x0_lo[b * P.n + d];
    hi = P.x0_hi[b * P.n + d];
  }
}

// symbolic_step's queue push + fold_overflow, hull branch (flowpipe_ct.hpp:
// 378-409, 347-348), for a non-square G0 (cl_reach): the fresh block
// diag(rad) joins the queue; if the queue overflows, the oldest block
// (columns [p0, p0 + na)) is boxed into the fresh block's diagonal and dropped.
// The oldest block's row sums are taken first and the fresh block is written
// after the shift, so rows never exceed nz columns: newest(i,i) = rad_i +
// row_abs_sum(oldest, i), the reference's one addition.  Lane i sweeps row i.
template <int RS>
__device__ __forceinline__ void push_fresh_fold(double* S, const Iv* erem, int na, int p0, int& nz, int& nq, int cap,
                                                int lane) {
  __syncwarp();
  const bool fold = nq + 1 > cap;
  double add = 0.0;
  if (fold && lane < na)
    for (int j = 0; j < na; ++j) add += fabs(S[lane * RS + p0 + j]);
  __syncwarp();
  if (fold) {
    for (int i = 0; i < na; ++i) {
      double v[NZC];
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        v[k] = (j >= p0 && j + na < nz) ? S[i * RS + j + na] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (j >= p0 && j < nz) S[i * RS + j] = v[k];
      }
    }
    nz -= na;
    nq -= 1;
  }
  __syncwarp();
  for (int i = 0; i < na; ++i) {
    const double ai = fold ? __shfl_sync(0xffffffffu, add, i) : 0.0;
    const double rad = (erem[i].hi - erem[i].lo) * 0.5;
#pragma unroll
    for (int k = 0; k < NZC; ++k) {
      const int j = lane + 32 * k;
      if (j >= nz && j < nz + na) S[i * RS + j] = (j - nz == i) ? (fold ? rad + ai : rad) : 0.0;
    }
  }
  nz += na;
  nq += 1;
  __syncwarp();
}

// symbolic_step + fold_overflow for a square G0 (ct_reach, flowpipe_ct.hpp:
// 317-346, 378-409): push the fresh block diag(rad); if the queue overflows
// (at most once per step: the queue held <= cap blocks), solve G0 X = Q_old
// by partial-pivot elimination (linalg.hpp:96-132: first maximum wins, pivot
// tolerance 1e-12, separate roundings), and if max_j rowabs(X)_j (1+1e-12) <= 1
// scale G0's columns by 1 + r_j and box the residual G0 X - Q_old into the
// fresh block's diagonal, else box Q_old itself (:347-348); then drop Q_old.
// Lane j < n + n holds column j of [G0 | Q_old] in registers; pivots and
// multipliers travel by shuffles.  Straight-line control flow throughout (no
// data-dependent loop exits), so the compiler keeps the warp provably
// converged for the shuffles of the surrounding flowpipe code.
__device__ __noinline__ void push_fresh_fold_square(double* S, const Iv* erem, int n, int& nz, int& nq, int cap,
                                                    double* scratch, int lane) {
  __syncwarp();
  for (int i = 0; i < n; ++i) {
    const double rad = (erem[i].hi - erem[i].lo) * 0.5;
#pragma unroll
    for (int k = 0; k < NZC; ++k) {
      const int j = lane + 32 * k;
      if (j >= nz && j < nz + n) S[i * NZP + j] = (j - nz == i) ? rad : 0.0;
    }
  }
  nz += n;
  nq += 1;
  __syncwarp();
  const bool fold = nq > cap;
  const int w = n, nc = 2 * n;
  const int off_new = nz - n;  // the fresh (newest) block
  double col[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) col[i] = (fold && lane < nc && i < n) ? S[i * NZP + lane] : 0.0;
  bool ok = fold;
  for (int kk = 0; kk < NA; ++kk) {
    const bool live = ok && kk < n;
    int piv = kk;
    double best = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const double v = fabs(col[i]);
      if (i == kk) best = v;
      if (i > kk && i < n && v > best) {
        best = v;
        piv = i;
      }
    }
    piv = __shfl_sync(0xffffffffu, piv, kk & 31);
    best = __shfl_sync(0xffffffffu, best, kk & 31);
    ok = ok && (!live || best > 1e-12);
    const bool go = live && ok;
    double vk = 0.0, vp = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (i == kk) vk = col[i];
      if (i == piv) vp = col[i];
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (go && piv != kk && i == kk) col[i] = vp;
      if (go && piv != kk && i == piv) col[i] = vk;
    }
    double akk = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i)
      if (i == kk) akk = col[i];
    double f[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) f[i] = (go && i > kk && i < n) ? __ddiv_rn(col[i], akk) : 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i) f[i] = __shfl_sync(0xffffffffu, f[i], kk & 31);
    double mk = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i)
      if (i == kk) mk = col[i];
    if (go && lane < nc && lane >= kk) {
#pragma unroll
      for (int i = 0; i < NA; ++i)
        if (i > kk && i < n) col[i] = sub(col[i], mul(f[i], mk));
    }
  }
  double* M = scratch;       // [n][nc] eliminated [U | B']
  double* X = M + n * nc;    // [n][w]
  double* E = X + n * w;     // [n][w]
  double* rr = E + n * w;    // [n]
  if (ok && lane < nc)
#pragma unroll
    for (int i = 0; i < NA; ++i)
      if (i < n) M[i * nc + lane] = col[i];
  __syncwarp();
  if (ok && lane >= n && lane < nc) {  // back substitution, lane n+j owns right-hand side j
    const int jc = lane - n;
    double x[NA];
#pragma unroll
    for (int i = NA - 1; i >= 0; --i) {
      if (i < n) {
        double a = col[i];
#pragma unroll
        for (int kk = i + 1; kk < NA; ++kk)
          if (kk < n) a = sub(a, mul(M[i * nc + kk], x[kk]));
        x[i] = __ddiv_rn(a, M[i * nc + i]);
        X[i * w + jc] = x[i];
      } else {
        x[i] = 0.0;
      }
    }
  }
  __syncwarp();
  if (ok && lane < n) {
    double s = 0.0;
    for (int j = 0; j < w; ++j) s = add(s, fabs(X[lane * w + j]));
    rr[lane] = mul(s, 1.0 + 1e-12);
  }
  __syncwarp();
  double worst = 0.0;
  for (int j = 0; ok && j < n; ++j) worst = smax(worst, rr[j]);
  const bool absorb = ok && worst <= 1.0;
  if (absorb && lane < w)  // residual e = G0 X - Q_old
    for (int i = 0; i < n; ++i) {
      double e = 0.0;
      for (int kk = 0; kk < n; ++kk) e = add(e, mul(S[i * NZP + kk], X[kk * w + lane]));
      E[i * w + lane] = sub(e, S[i * NZP + n + lane]);
    }
  __syncwarp();
  if (fold && lane < n) {
    double s = 0.0;
    if (absorb) {
      const double sc = add(1.0, rr[lane]);
      for (int i = 0; i < n; ++i) S[i * NZP + lane] = mul(S[i * NZP + lane], sc);
      for (int j = 0; j < w; ++j) s = add(s, fabs(E[lane * w + j]));
      s = mul(s, 1.0 + 1e-12);
    } else {
      for (int j = 0; j < w; ++j) s = add(s, fabs(S[lane * NZP + n + j]));
    }
    S[lane * NZP + off_new + lane] = add(S[lane * NZP + off_new + lane], s);
  }
  __syncwarp();
  // drop Q_old: columns [2n, nz) -> [n, nz - n)
  if (fold) {
    for (int i = 0; i < n; ++i) {
      double v[NZC];
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        v[k] = (j >= n && j + n < nz) ? S[i * NZP + j + n] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (j >= n && j < nz) S[i * NZP + j] = v[k];
      }
    }
    nz -= n;
    nq -= 1;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Flowpipe steps, one warp per sub-box: k_atomic steps of one control
// interval (cl_reach, SQUARE = false) or the whole horizon (ct_reach, SQUARE =
// true).  Two instantiations: the square fold's shuffles otherwise cost the
// cl_reach kernel the compiler's proof of warp convergence (collective
// shuffle fallbacks everywhere, +35 % time).
#ifndef RB_CT_FLOW_MINB
#define RB_CT_FLOW_MINB 10  // compact layout: 10 sub-boxes per SM -> 3 warps per scheduler: <= 168 registers (16 K per SMSP)
#endif
template <bool SQUARE, bool CMP>
__global__ void __launch_bounds__(32, CMP ? RB_CT_FLOW_MINB : 1) ct_flow_kernel(const CTParams Pm) {
  extern __shared__ __align__(16) unsigned char ct_smem[];
  FlowSmem& W = *reinterpret_cast<FlowSmem*>(ct_smem);
  static_assert(!(SQUARE && CMP), "the compact layout is cl_reach's");
  constexpr int RS = CMP ? kRowC : NZP;  // shared-memory row stride (the HBM state keeps NZP)
  double* coef = flow_coef<CMP>(W);
  const long long b = blockIdx.x;
  if (b >= Pm.B) return;
  const int lane = threadIdx.x;
  const int na = SQUARE ? Pm.na : NA, p0 = Pm.n;  // cl_reach: the augmented quadrotor, 16 rows
  const bool init = Pm.ct && Pm.ci == 0;
  int* meta = Pm.st_meta + b * 4;
  int nq = 0, status = CT_OK, fstep = -1, nboxes = 0;
  if (!init) {
    nq = meta[0];
    status = meta[1];
    fstep = meta[2];
    nboxes = meta[3];
  }
  const bool last = (Pm.ci + 1 == Pm.ctl_steps);
  if (status != CT_OK) {
    if (last && lane == 0) finalize(Pm, b, nboxes, status, fstep);
    return;
  }
  const double h = Pm.h;
  const int cap = Pm.window > 0 ? Pm.window : 1;
  int nz = p0 + nq * Pm.bw;
  double* gM = Pm.st_M + static_cast<size_t>(b) * NA * NZP;
  Side sd;
  if constexpr (CMP) {
    unsigned char* g = Pm.side + static_cast<size_t>(b) * kSideBytes;
    sd = Side{reinterpret_cast<Iv*>(g), reinterpret_cast<Iv*>(g) + NA, reinterpret_cast<Iv*>(g) + 2 * NA,
              reinterpret_cast<Iv*>(g) + 3 * NA, reinterpret_cast<double2*>(g + 4 * NA * sizeof(Iv))};
  } else {
    sd = Side{W.erem_s, W.i0_s, W.i1_s, W.nx_s, W.fc_s};
  }
  // ---- the field program, its constants and the row layout
  int npb = 0;
  for (int i = 0; i < na; ++i) npb += (Pm.bzsrc[i] == -1);
  const int off_zero = CMP ? kNoRow : na * RS, off_pbz = na * RS + (CMP ? 0 : RS), off_taz = off_pbz + npb * RS,
            off_tbz = off_taz + NTF * RS, coef_end = off_tbz + NTF * RS;
  if (lane < kMaxKc) W.kc[lane] = Pm.kc[lane];
  if (lane == 0) {
    W.na = na;
    W.off_zero = off_zero;
    W.off_pbz = off_pbz;
    W.off_taz = off_taz;
    W.off_tbz = off_tbz;
    int q = 0;
    for (int i = 0; i < na; ++i) {
      const int src = Pm.bzsrc[i];
      W.own[i] = (src == -1);
      W.pbz[i] = (src == -1) ? off_pbz + (q++) * RS : (src == -2) ? off_zero : src * RS;
    }
    for (int i = 0; i < 8; ++i) W.wid[i] = Pm.bw;
  }
  for (int s = lane; s < (CMP ? NA : NSLOT); s += 32) {  // the compact header holds the P slots only
    Slot& d = W.D[s];
    d.s1 = 1.0;
    d.s2 = 1.0;
    d.view = 0;
    d.az = (s < SLOT_T) ? s * RS : (s < SLOT_V) ? off_taz + (s - SLOT_T) * RS : off_zero;
    d.bz = (s < SLOT_V && s >= SLOT_T) ? off_tbz + (s - SLOT_T) * RS : off_zero;
  }
  // ---- the state: from X0 (ct_reach, init_symbolic_state, flowpipe_ct.hpp:302-309) or HBM
  for (int t = lane; t < coef_end; t += 32) coef[t] = 0.0;
  __syncwarp();
  for (int s = lane; s < NA; s += 32)
    if (s < na) W.D[s].bz = W.pbz[s];
  if (init) {
    double lo = 0.0, hi = 0.0;
    if (lane < na) {
      x0_box(Pm, b, lane, lo, hi);
      W.sc[lane] = (lo + hi) * 0.5;
      coef[lane * RS + lane] = (hi - lo) * 0.5;
      emit_box(Pm, b, 0, na, lane, lo, hi);  // box 0 is X0 itself (flowpipe_ct.hpp:433)
    }
    nboxes = 1;
  } else {
    for (int i = 0; i < na; ++i)
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (j < nz) coef[i * RS + j] = gM[i * NZP + j];
      }
    if (lane < na) W.sc[lane] = Pm.st_c[b * NA + lane];
  }
  __syncwarp();

  Lane L;
  L.lane = lane;
  L.h = h;
  for (int step = 0; step < Pm.K && status == CT_OK; ++step) {
    const int gstep = Pm.ci * Pm.K + step;
#pragma unroll
    for (int k = 0; k < NZC; ++k) L.act[k] = (lane + 32 * k) < nz;
    // seed rows: abs_z (cached: the Picard rows share their z columns)
    {
      double v[NA];
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        v[i] = 0.0;
#pragma unroll
        for (int k = 0; k < NZC; ++k)
          if (i < na && L.act[k]) v[i] += fabs(coef[i * RS + lane + 32 * k]);
      }
      const double sum = wsum16_rows(v, lane);
      if ((lane & 1) == 0 && row_of_wsum16(lane) < na) W.ssz[row_of_wsum16(lane)] = sum;
      __syncwarp();
    }
    // poly_picard (flowpipe_ct.hpp:126-139): g_0 = seed (bz = 0, at = 0, rem = 0);
    // aliased rows are never read before their first update
    for (int i = 0; i < na; ++i) {
      if (W.own[i])
#pragma unroll
        for (int k = 0; k < NZC; ++k)
          if (L.act[k]) coef[W.pbz[i] + lane + 32 * k] = 0.0;
      set_scalars(W.D[i], W.sc[i], 0.0, Iv{0.0, 0.0}, W.ssz[i], 0.0);
    }
    bool thrown = false;
    auto full_field = [&](int mode) {
      if constexpr (CMP) {
        return quad_full<false, true>(W, sd, mode, L, gM);
      } else {
        if (Pm.fast_prog == 1) return quad_full<false>(W, sd, mode, L, gM);
        if (Pm.fast_prog == 2) return quad_full<true>(W, sd, mode, L, gM);
        return run_field(W, Pm.prog, mode, L, gM);
      }
    };
    for (int it = 0; it < Pm.order && !thrown; ++it) {
      thrown = full_field(MODE_PICARD);
      __syncwarp();
    }
    int fail = thrown ? CT_TME_INV : CT_OK;
    // the per-row checks and updates of remainder_picard run lane-parallel (lane i: row i < na <= 16)
    const bool row = lane < na;
    if (fail == CT_OK && __any_sync(0xffffffffu, row && !isfinite(W.D[lane].c))) fail = CT_PICARD;
    // remainder_picard (flowpipe_ct.hpp:144-276)
    bool cached = false;  // this step's full replay has run (FlowSmem::fc, the endpoint rows in HBM)
    int nrec = 0;  // 0: nothing recorded yet; 1: quad_fast's constants recorded (the temporaries' rows)
    auto fast_field = [&](int mode) {
      bool t;
      if constexpr (CMP) {
        t = nrec ? quad_fast<false, true, true>(W, sd, mode, h, false) : quad_fast<false, false, true>(W, sd, mode, h, true);
      } else {
        if (Pm.fast_prog == 1)
          t = nrec ? quad_fast<false, true>(W, sd, mode, h, false) : quad_fast<false, false>(W, sd, mode, h, true);
        else if (Pm.fast_prog == 2)
          t = nrec ? quad_fast<true, true>(W, sd, mode, h, false) : quad_fast<true, false>(W, sd, mode, h, true);
        else
          t = run_field(W, Pm.prog, mode, L, gM);
      }
      nrec = 1;
      return t;
    };
    auto replay = [&](const Iv* cand) {
      if (row) {
        W.D[lane].rlo = cand[lane].lo;
        W.D[lane].rhi = cand[lane].hi;
      }
      __syncwarp();
      const bool t = cached ? fast_field(MODE_REPLAY_FAST) : full_field(MODE_REPLAY);
      __syncwarp();  // lane 0's cache stores before the next replay's reads
      cached = true;
      return t;
    };
    auto finite_box = [&](const Iv* x) { return __all_sync(0xffffffffu, !row || ifin(x[lane])); };
    auto subset = [&](const Iv* in, const Iv* out) {
      return __all_sync(0xffffffffu, !row || (out[lane].lo <= in[lane].lo && in[lane].hi <= out[lane].hi));
    };
    if (fail == CT_OK) {
      if (row) {
        sd.i0[lane] = Iv{-Pm.eps, Pm.eps};
        sd.i1[lane] = Iv{0.0, 0.0};
      }
      bool accepted = false;
      for (int attempt = 0; attempt <= Pm.maxe; ++attempt) {
        const bool threw = replay(sd.i0);
        if (!threw && row) sd.i1[lane] = sd.nx[lane];
        if (!threw && finite_box(sd.i1) && subset(sd.i1, sd.i0)) {
          accepted = true;
          break;
        }
        if (row) {  // per-dimension adaptive enlargement (:178-182)
          const Iv ind = threw ? Iv{0.0, 0.0} : sd.i1[lane];
          const Iv cur = sd.i0[lane];
          const Iv hull = (ind.lo <= ind.hi) ? Iv{smin(cur.lo, ind.lo), smax(cur.hi, ind.hi)} : cur;
          const double mid = (hull.lo + hull.hi) * 0.5, rad = (hull.hi - hull.lo) * 0.5 * Pm.enl;
          sd.i0[lane] = Iv{mid - rad, mid + rad};
        }
        __syncwarp();
      }
      __syncwarp();
      if (!accepted) fail = CT_REMAINDER;
    }
    if (fail == CT_OK) {
      for (int round = 0; round < Pm.refine; ++round) {  // shrink (:214-223)
        if (replay(sd.i1)) break;
        if (!(finite_box(sd.nx) && subset(sd.nx, sd.i1))) break;
        if (row) sd.i1[lane] = sd.nx[lane];
      }
      // endpoint by exact integration at tau = h (:236-263) into the HBM state rows
      if (row) {
        W.D[lane].rlo = sd.i1[lane].lo;
        W.D[lane].rhi = sd.i1[lane].hi;
      }
      __syncwarp();
      const bool threw = fast_field(MODE_ENDPOINT);
      const bool exact_ok = !threw && finite_box(sd.erem) && __all_sync(0xffffffffu, !row || isfinite(W.ec[lane]));
      // tm_eval_interval(segment, [0, h]) (taylor_model.hpp:73-97), before S changes; lane i: row i
      const int kbox = 1 + gstep;
      double blo = 0.0, bhi = 0.0;
      if (row) {
        const Slot& p = W.D[lane];
        Iv acc{p.c - p.sz, p.c + p.sz};
        acc = iadd(acc, iscale(p.at, Iv{0.0, h}));
        const double tau_mag = smax(0.0, h);
        acc = iadd(acc, Iv{-p.sb * tau_mag, p.sb * tau_mag});
        acc = iadd(acc, sd.i1[lane]);
        blo = acc.lo;
        bhi = acc.hi;
      }
      const bool fin = __all_sync(0xffffffffu, !row || ifin(Iv{blo, bhi}));
      if (row) emit_box(Pm, b, kbox, na, lane, blo, bhi);
      nboxes = kbox + 1;
      // new generator rows: the exact endpoint (HBM, L2-resident) or the
      // fallback p_k(h) = seed + B h (:264-274), via HBM so aliased bz rows
      // are read before any seed row changes
      if (!exact_ok) {
        for (int i = 0; i < na; ++i) {
#pragma unroll
          for (int k = 0; k < NZC; ++k) {
            if (!L.act[k]) continue;
            const int j = lane + 32 * k;
            gM[i * NZP + j] = coef[i * RS + j] + rowv(coef, W.pbz[i], j) * h;
          }
          W.ec[i] = W.D[i].c + W.D[i].at * h;
          sd.erem[i] = sd.i1[i];
        }
      }
      for (int i = 0; i < na; ++i)
#pragma unroll
        for (int k = 0; k < NZC; ++k) {
          if (!L.act[k]) continue;
          const int j = lane + 32 * k;
          coef[i * RS + j] = gM[i * NZP + j];
        }
      if (!fin) {
        fail = CT_BOX;
      } else {
        // symbolic_step (flowpipe_ct.hpp:378-409)
        double c_new = 0.0;
        if (lane < na) c_new = W.ec[lane] + (sd.erem[lane].lo + sd.erem[lane].hi) * 0.5;
        if constexpr (SQUARE)
          push_fresh_fold_square(coef, sd.erem, na, nz, nq, cap, coef + off_pbz, lane);
        else
          push_fresh_fold<RS>(coef, sd.erem, na, p0, nz, nq, cap, lane);
        if (lane < na) W.sc[lane] = c_new;
        __syncwarp();
      }
    }
    if (fail != CT_OK) {
      status = fail;
      fstep = gstep;
    }
  }
  // state out
  __syncwarp();
  for (int i = 0; i < na; ++i)
#pragma unroll
    for (int k = 0; k < NZC; ++k) {
      const int j = lane + 32 * k;
      if (j < NZP) gM[i * NZP + j] = (j < nz) ? coef[i * RS + j] : 0.0;
    }
  if (lane < na) Pm.st_c[b * NA + lane] = W.sc[lane];
  if (lane == 0) {
    meta[0] = nq;
    meta[1] = status;
    meta[2] = fstep;
    meta[3] = nboxes;
    if (last || status != CT_OK) finalize(Pm, b, nboxes, status, fstep);
  }
}

// ---------------------------------------------------------------------------
// Controller certification + stacking (closed_loop.hpp:89-155), one warp per
// sub-box.  Weights are read from the uploaded blob (W row-major, W^T) through
// L1/L2: the controller is small and certified once per control interval.
// Per warp: this struct, then the preactivation boxes of the controller's
// hidden layers, [L - 1][CW][2] (sized by the host).  CW is the widest
// controller layer rounded up to 64 or 128: the C2 controller (3 x 64) takes
// 18.8 KB per warp -> 12 sub-boxes per SM (8 with 128-wide buffers).
template <int CW>
struct __align__(16) CtlSmem {
  static constexpr int LA = CW > NZP ? CW : NZP;  // Lambda rows double as the 4 x nzx Lambda_z scratch
  double xA[NX * LDX];           // state TM rows (n x nzx), stride LDX
  double xc[NX];
  double hb[2][CW][2];           // IBP boxes
  double lam[2][4][LA];          // Lambda (n_o x width), double buffered
  double bf0[CW];                // frozen first-layer bias
  double blo[4], bup[4];
  double uc[4];
  Iv urem[4];
};
template <int CW>
__host__ __device__ constexpr size_t ctl_warp_bytes(int layers) {
  return sizeof(CtlSmem<CW>) + static_cast<size_t>(layers - 1) * CW * 2 * sizeof(double);
}

constexpr int kCtlWarps = 4;
constexpr int kCtlPrefetch = 16;  // controller weights loaded a chunk ahead of their accumulation chain
__device__ __forceinline__ void ctl_chunk(double (&v)[kCtlPrefetch], const double* base, size_t ld, int j0, int n) {
#pragma unroll
  for (int q = 0; q < kCtlPrefetch; ++q) v[q] = (j0 + q < n) ? __ldg(base + static_cast<size_t>(j0 + q) * ld) : 0.0;
}

__device__ __forceinline__ void relax_tanh_or_relu(int act, double l, double u, double& s, double& li, double& ui) {
  relax(act, l, u, s, li, ui);
}

template <int CW>
__global__ void __launch_bounds__(32 * kCtlWarps) ct_ctl_kernel(const CTParams Pm) {
  extern __shared__ __align__(16) unsigned char ct_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CtlSmem<CW>& W = *reinterpret_cast<CtlSmem<CW>*>(ct_smem + warp * ctl_warp_bytes<CW>(Pm.ctl.L));
  double* pre = reinterpret_cast<double*>(&W + 1);  // [L - 1][CW][2]
  constexpr int LA = CtlSmem<CW>::LA;
  const long long b = static_cast<long long>(blockIdx.x) * kCtlWarps + warp;
  if (b >= Pm.B) return;
  const int n = Pm.n, l = Pm.l;
  const int cap = Pm.window > 0 ? Pm.window : 1;
  int* meta = Pm.st_meta + b * 4;
  int nq = 0, status = CT_OK, fstep = -1, nboxes = 0;
  if (Pm.ci > 0) {
    nq = meta[0];
    status = meta[1];
    fstep = meta[2];
    nboxes = meta[3];
    if (status != CT_OK) return;
  }
  const int gstep = Pm.ci * Pm.K;
  double* gM = Pm.st_M + static_cast<size_t>(b) * NA * NZP;
  double* gc = Pm.st_c + b * NA;

  // ---- x_tm: build_linear_tm(X0) (taylor_model.hpp:53-64), the boundary
  // state TM (closed_loop.hpp:51-69) or the intervalized box (:93-97)
  int nzx, nbw;
  bool box_tm = (Pm.ci == 0) || Pm.intervalize;
  if (box_tm) {
    double lo = 0.0, hi = 0.0;
    if (lane < n) {
      if (Pm.ci == 0) {
        if (Pm.split) {
          long long p = Pm.part_begin + b;
          for (int d = n - 1; d >= 0; --d) {
            const int k = Pm.counts[d];
            const int i = static_cast<int>(p % k);
            p /= k;
            if (d == lane) {
              const double xl = Pm.sx_lo[d], xh = Pm.sx_hi[d];
              lo = (i == 0) ? xl : xl + (xh - xl) * (static_cast<double>(i) / k);
              hi = (i + 1 == k) ? xh : xl + (xh - xl) * (static_cast<double>(i + 1) / k);
            }
          }
        } else {
          lo = Pm.x0_lo[b * n + lane];
          hi = Pm.x0_hi[b * n + lane];
        }
      } else {  // symbolic_box of the state rows (flowpipe_ct.hpp:413-424)
        const int nz = n + nq * NA;
        double r = 0.0;
        for (int j = 0; j < n; ++j) r += fabs(gM[lane * NZP + j]);
        for (int q = 0; q < nq; ++q) {
          double rq = 0.0;
          for (int j = 0; j < NA; ++j) rq += fabs(gM[lane * NZP + n + q * NA + j]);
          r += rq;
        }
        (void)nz;
        lo = gc[lane] - r;
        hi = gc[lane] + r;
      }
    }
    const bool xfin = __all_sync(0xffffffffu, lane >= n || (isfinite(lo) && isfinite(hi)));
    if (!xfin) {  // build_linear_tm throws; the exception escapes cl_reach
      if (lane == 0) {
        meta[1] = CT_OTHER;
        meta[2] = 0;
        meta[3] = 0;
      }
      return;
    }
    nzx = n;
    nbw = 0;
    for (int i = 0; i < n; ++i)
      for (int j = lane; j < n; j += 32) W.xA[i * LDX + j] = 0.0;
    __syncwarp();
    if (lane < n) {
      W.xc[lane] = (lo + hi) * 0.5;
      W.xA[lane * LDX + lane] = (hi - lo) * 0.5;
    }
  } else {
    nzx = n + nq * NA;
    nbw = nq;
    double v[NX][NZC];  // every load in flight before the first store (n == NX for cl_reach)
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        v[i][k] = (i < n && j < nzx) ? gM[i * NZP + j] : 0.0;
      }
#pragma unroll
    for (int i = 0; i < NX; ++i)
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (i < n && j < nzx) W.xA[i * LDX + j] = v[i][k];
      }
    if (lane < n) W.xc[lane] = gc[lane];
  }
  __syncwarp();

  // ---- ctl_crown (neural.hpp:418-424): freeze the reference into the
  // first-layer bias (freeze_trailing_inputs, :398-413), certify_tm_input.
  const DevNet& N = Pm.ctl;
  const int Lc = N.L;
  const double* blob = N.blob;
  for (int u = lane; u < N.dims[1]; u += 32) {
    double bb = blob[N.b_off[0] + u];
    for (int j = 0; j < Pm.ref_dim; ++j)
      bb = bb + blob[N.w_off[0] + static_cast<size_t>(u) * N.ldw[0] + n + j] * Pm.y_ref[Pm.ci * Pm.ref_dim + j];
    W.bf0[u] = bb;
  }
  // prepend-layer IBP (neural.hpp:360-373, interval.hpp:284-295): lane = state row
  if (lane < n) {
    double lo = 0.0, hi = 0.0;
    for (int j = 0; j < nzx; ++j) {
      const double a = W.xA[lane * LDX + j];
      lo = lo + ((a >= 0.0) ? -a : a);
      hi = hi + ((a >= 0.0) ? a : -a);
    }
    W.hb[0][lane][0] = lo + W.xc[lane];
    W.hb[0][lane][1] = hi + W.xc[lane];
  }
  __syncwarp();
  // hidden-layer IBP (neural.hpp:243-257): lane = output unit, W^T rows
  int cur = 0;
  for (int t = 0; t + 1 < Lc; ++t) {
    const int rows = N.dims[t], width = N.dims[t + 1];
    const int in_cols = (t == 0) ? n : rows;
    for (int u = lane; u < width; u += 32) {
      double lo = 0.0, hi = 0.0;
      const double* wt = blob + N.wt_off[t] + u;
      const size_t ldt = N.ldt[t];
      double wv[kCtlPrefetch];
      ctl_chunk(wv, wt, ldt, 0, in_cols);
      for (int j0 = 0; j0 < in_cols; j0 += kCtlPrefetch) {  // the next chunk's weights in flight (L2 latency)
        double wn[kCtlPrefetch];
        ctl_chunk(wn, wt, ldt, j0 + kCtlPrefetch, in_cols);
#pragma unroll
        for (int q = 0; q < kCtlPrefetch; ++q) {
          if (j0 + q >= in_cols) break;
          const double w = wv[q];
          const double xl = W.hb[cur][j0 + q][0], xh = W.hb[cur][j0 + q][1];
          lo = lo + ((w >= 0.0) ? w * xl : w * xh);
          hi = hi + ((w >= 0.0) ? w * xh : w * xl);
        }
#pragma unroll
        for (int q = 0; q < kCtlPrefetch; ++q) wv[q] = wn[q];
      }
      const double bias = (t == 0) ? W.bf0[u] : blob[N.b_off[t] + u];
      lo = lo + bias;
      hi = hi + bias;
      pre[(t * CW + u) * 2] = lo;
      pre[(t * CW + u) * 2 + 1] = hi;
      W.hb[cur ^ 1][u][0] = act_apply(N.acts[t], lo);
      W.hb[cur ^ 1][u][1] = act_apply(N.acts[t], hi);
    }
    cur ^= 1;
    __syncwarp();
  }
  // CROWN backward (neural.hpp:290-335) on the wide net [prepend; ctl layers]
  const int no = l;
  int lb = 0;
  const int wout = N.dims[Lc - 1];
  // output layer (identity): Lambda = I, shift = b_out, Lambda = W_out
  if (lane < no) {
    W.blo[lane] = blob[N.b_off[Lc - 1] + lane];
    W.bup[lane] = W.blo[lane];
  }
  for (int i = 0; i < no; ++i)
    for (int j = lane; j < wout; j += 32) W.lam[lb][i][j] = blob[N.w_off[Lc - 1] + static_cast<size_t>(i) * N.ldw[Lc - 1] + j];
  __syncwarp();
  bool bad = false;
  for (int t = Lc - 2; t >= 0; --t) {
    const int width = N.dims[t + 1];
    const int cols = (t == 0) ? n : N.dims[t];
    // relax_activation (neural.hpp:166-227) per unit; non-finite -> throw
    for (int u = lane; u < width; u += 32) {
      double s, li, ui;
      const double pl = pre[(t * CW + u) * 2], ph = pre[(t * CW + u) * 2 + 1];
      if (!(isfinite(pl) && isfinite(ph))) {
        bad = true;
        s = li = ui = 0.0;
      } else {
        relax(N.acts[t], pl, ph, s, li, ui);
      }
      pre[(t * CW + u) * 2] = s;
      W.hb[0][u][0] = li;
      W.hb[0][u][1] = ui;
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad) break;
    __syncwarp();
    // intercept chains (sequential in j, lane = output row i), slope scaling
    if (lane < no) {
      double bl = W.blo[lane], bu = W.bup[lane];
      for (int j = 0; j < width; ++j) {
        const double aij = W.lam[lb][lane][j];
        const double li = W.hb[0][j][0], ui = W.hb[0][j][1];
        if (aij >= 0.0) {
          bl = bl + aij * li;
          bu = bu + aij * ui;
        } else {
          bl = bl + aij * ui;
          bu = bu + aij * li;
        }
        W.lam[lb][lane][j] = aij * pre[(t * CW + j) * 2];
      }
      // shift = Lambda . b (linalg.hpp:40-51), b += shift
      const double* bias = (t == 0) ? W.bf0 : blob + N.b_off[t];
      double sh = 0.0;
      for (int j = 0; j < width; ++j) sh = sh + W.lam[lb][lane][j] * bias[j];
      W.blo[lane] = bl + sh;
      W.bup[lane] = bu + sh;
    }
    __syncwarp();
    // Lambda = Lambda . W_t (linalg.hpp:53-63, i-k-j order): lane = column
    for (int jc = lane; jc < cols; jc += 32) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const double* wc = blob + N.w_off[t] + jc;
      const size_t ldw = N.ldw[t];
      double wv[kCtlPrefetch];
      ctl_chunk(wv, wc, ldw, 0, width);
      for (int k0 = 0; k0 < width; k0 += kCtlPrefetch) {
        double wn[kCtlPrefetch];
        ctl_chunk(wn, wc, ldw, k0 + kCtlPrefetch, width);
#pragma unroll
        for (int q = 0; q < kCtlPrefetch; ++q) {
          if (k0 + q >= width) break;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < no) acc[i] = acc[i] + W.lam[lb][i][k0 + q] * wv[q];
        }
#pragma unroll
        for (int q = 0; q < kCtlPrefetch; ++q) wv[q] = wn[q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < no) W.lam[lb ^ 1][i][jc] = acc[i];
    }
    lb ^= 1;
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) {
      meta[0] = nq;
      meta[1] = CT_CTL_FAILED;
      meta[2] = gstep;
      meta[3] = nboxes;
    }
    return;
  }
  // prepend layer (identity, W = [A | I], b = c): shift = Lambda . c, Lambda_z = Lambda . A
  if (lane < no) {
    double sh = 0.0;
    for (int k = 0; k < n; ++k) sh = sh + W.lam[lb][lane][k] * W.xc[k];
    const double bl = W.blo[lane] + sh, bu = W.bup[lane] + sh;
    // tail (neural.hpp:383-391); the r-block adds iv_scale(., [0, 0])
    const double mid = (bl + bu) * 0.5;
    W.uc[lane] = mid;
    W.urem[lane] = Iv{bl - mid, bu - mid};
  }
  // stacked state rows: x rows then u rows; columns [0, nzx) then the fresh block
  double* S = W.lam[lb ^ 1][0];  // scratch for Lambda_z (4 x nzx)
  for (int jc = lane; jc < nzx; jc += 32) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < n; ++k) {
      const double a = W.xA[k * LDX + jc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < no) acc[i] = acc[i] + W.lam[lb][i][k] * a;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < no) S[i * LA + jc] = acc[i];
  }
  __syncwarp();
  bool ufin = true;
  for (int i = 0; i < no; ++i) ufin = ufin && ifin(W.urem[i]);
  if (!ufin) {
    if (lane == 0) {
      meta[0] = nq;
      meta[1] = CT_CTL_DIVERGED;
      meta[2] = gstep;
      meta[3] = nboxes;
    }
    return;
  }
  // ---- stacking (closed_loop.hpp:122-153) into global memory: rows [x; u]
  // over columns [0, nzx), then the fresh diagonal block of the remainder
  // radii.  If the queue overflows, fold_overflow's hull branch
  // (flowpipe_ct.hpp:347-348; G0 = (n + l) x n is never square) boxes the
  // oldest block (columns [n, n + NA)) into the fresh block's diagonal and
  // drops it, so the rows are written in their folded layout directly.
  auto stacked = [&](int d, int j) { return (d < n) ? W.xA[d * LDX + j] : S[(d - n) * LA + j]; };
  const bool fold = nbw + 1 > cap;
  const int nz_keep = fold ? nzx - NA : nzx;
  const int nqn = fold ? nbw : nbw + 1;
  const int nz = nz_keep + NA;
  double add = 0.0;
  if (fold && lane < NA)
    for (int j = 0; j < NA; ++j) add += fabs(stacked(lane, n + j));
  for (int d = 0; d < NA; ++d) {
    const double ad = fold ? __shfl_sync(0xffffffffu, add, d) : 0.0;
    const double rad = (d < n) ? (0.0 - 0.0) * 0.5 : (W.urem[d - n].hi - W.urem[d - n].lo) * 0.5;
    for (int j = lane; j < NZP; j += 32) {
      double v = 0.0;
      if (j < nz_keep) {
        v = stacked(d, (fold && j >= n) ? j + NA : j);
      } else if (j - nz_keep == d) {
        v = fold ? rad + ad : rad;
      }
      gM[d * NZP + j] = v;
    }
  }
  if (lane < NA) gc[lane] = (lane < n) ? W.xc[lane] + (0.0 + 0.0) * 0.5
                                       : W.uc[lane - n] + (W.urem[lane - n].lo + W.urem[lane - n].hi) * 0.5;
  __syncwarp();
  (void)nz;
  // box 0 = symbolic_box of the first augmented state (closed_loop.hpp:155)
  if (Pm.ci == 0) {
    __syncwarp();
    if (lane < NA) {
      double r = 0.0;
      for (int j = 0; j < n; ++j) r += fabs(gM[lane * NZP + j]);
      for (int q = 0; q < nqn; ++q) {
        double rq = 0.0;
        for (int j = 0; j < NA; ++j) rq += fabs(gM[lane * NZP + n + q * NA + j]);
        r += rq;
      }
      const double c = gc[lane];
      emit_box(Pm, b, 0, NA, lane, c - r, c + r);
    }
    nboxes = 1;
  }
  if (lane == 0) {
    meta[0] = nqn;
    meta[1] = CT_OK;
    meta[2] = -1;
    meta[3] = nboxes;
  }
}

}  // namespace ct
}  // namespace rb
