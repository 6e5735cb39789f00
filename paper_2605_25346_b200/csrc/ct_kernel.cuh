// Continuous-time closed-loop reachability kernels for B200 (sm_100a):
// cl_reach (closed_loop.hpp:76-182) with the quadrotor plant augmented by
// udot = 0 rows (make_augmented_field, fields.hpp:96-128; quadrotor_ode,
// systems.hpp:22-64) under a neural (tanh / ReLU) controller.
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
// lane L owns generator columns L, L+32, L+64 of az and bz, so every TMExpr
// operation (products with excess folding, reciprocal, sin / cos,
// integration) is a per-lane FP64 update of three coefficient slots plus
// warp-uniform scalar interval arithmetic; the abs-sums the remainder bounds
// need (abs_z / abs_b) are butterfly shuffle reductions, computed once when a
// row is produced and cached next to it.  Lanes only ever touch their own
// coefficient slots, so the algebra needs no warp barriers.
//
// Numerics: the reference's operation order inside every TMExpr operation;
// the abs-sums are tree reductions (the reference sums sequentially) and libm
// is CUDA's (sin / cos / tanh), so results agree with the reference to
// rounding (tests: <= 1e-9 relative), not bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dt_common.cuh"
#include "dt_kernel.cuh"

namespace rb {
namespace ct {

constexpr int NX = 12;      // quadrotor state
constexpr int NA = 16;      // augmented (x, u)
constexpr int NZC = 3;      // generator slots per lane
constexpr int NZP = 32 * NZC;  // generator columns per row (nz <= 96)
constexpr int NT = 10;      // temporary rows of one field evaluation
constexpr int LDS = NZP + 1;   // state row stride in shared memory (odd: conflict-free row sweeps)
constexpr int kMaxCtlW = 128;  // widest controller layer (and input dim)
constexpr int LDX = NZP + 1;

// REACH_TUBE_* codes
enum : int { CT_OK = 0, CT_CTL_FAILED = 4, CT_CTL_DIVERGED = 5, CT_REMAINDER = 6, CT_PICARD = 7, CT_TME_INV = 8,
             CT_BOX = 3, CT_OTHER = 99 };

struct CTParams {
  int B, n, l, K, window, order, refine, maxe, intervalize, ref_dim, ci, ctl_steps;
  double h, eps, enl;
  double prm[8];
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
__device__ __forceinline__ Iv iv(double lo, double hi) { return Iv{lo, hi}; }
__device__ __forceinline__ Iv iadd(Iv a, Iv b) { return Iv{a.lo + b.lo, a.hi + b.hi}; }
__device__ __forceinline__ Iv isub(Iv a, Iv b) { return Iv{a.lo - b.hi, a.hi - b.lo}; }
__device__ __forceinline__ Iv imul(Iv a, Iv b) {
  const double p1 = a.lo * b.lo, p2 = a.lo * b.hi, p3 = a.hi * b.lo, p4 = a.hi * b.hi;
  return Iv{smin(smin(p1, p2), smin(p3, p4)), smax(smax(p1, p2), smax(p3, p4))};
}
__device__ __forceinline__ Iv iscale(double a, Iv x) {
  return (a >= 0.0) ? Iv{a * x.lo, a * x.hi} : Iv{a * x.hi, a * x.lo};
}
__device__ __forceinline__ bool ifin(Iv x) { return isfinite(x.lo) && isfinite(x.hi); }

__device__ __forceinline__ void wsum2(double& a, double& b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}
__device__ __forceinline__ double wsum(double a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

// ---------------------------------------------------------------------------
// One TMExpr row in shared memory.  Scalars are warp-uniform: every lane
// writes the same value, so a lane always reads back its own store.
struct Row {
  double az[NZP];
  double bz[NZP];
  double c, at, rlo, rhi;
  double sz, sb;  // cached abs_z / abs_b (taylor_model.hpp:213-224)
  double pad[2];
};

struct Lane {
  int lane;
  double h;
  bool act[NZC];  // slot lane + 32 k < nz
};

// poly_range (taylor_model.hpp:227-235) from the cached sums.
__device__ __forceinline__ Iv poly_range(double c, double sz, double at, double sb, double h) {
  Iv r{c - sz, c + sz};
  r = iadd(r, imul(Iv{0.0, h}, Iv{at, at}));
  const double br = sb * h;
  return iadd(r, Iv{-br, br});
}
__device__ __forceinline__ Iv total_range(const Row& u, double h) {
  return iadd(poly_range(u.c, u.sz, u.at, u.sb, h), Iv{u.rlo, u.rhi});
}

__device__ __forceinline__ void put_scalars(Row& r, double c, double at, Iv rem, double sz, double sb) {
  r.c = c;
  r.at = at;
  r.rlo = rem.lo;
  r.rhi = rem.hi;
  r.sz = sz;
  r.sb = sb;
}

// operator* (taylor_model.hpp:325-360).  r may alias u or v.
__device__ __forceinline__ void tm_mul(Row& r, const Row& u, const Row& v, const Lane& L) {
  const double h = L.h;
  const double uc = u.c, vc = v.c, uat = u.at, vat = v.at;
  const double au = u.sz, av = v.sz, bu = u.sb, bv = v.sb;
  const Iv ur{u.rlo, u.rhi}, vr{v.rlo, v.rhi};
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    const double ua = u.az[j], ub = u.bz[j], va = v.az[j], vb = v.bz[j];
    const double ra = uc * va + vc * ua;
    const double rb = uc * vb + vc * ub + uat * va + vat * ua;
    r.az[j] = ra;
    r.bz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  double sym = au * av;
  sym += (au * bv + av * bu) * h;
  sym += bu * bv * h * h;
  sym += (fabs(uat) * bv + fabs(vat) * bu) * h * h;
  Iv rem{-sym, sym};
  const double tt = uat * vat;
  rem = iadd(rem, imul(Iv{0.0, h * h}, Iv{tt, tt}));
  const Iv pu = poly_range(uc, au, uat, bu, h), pv = poly_range(vc, av, vat, bv, h);
  rem = iadd(rem, imul(pu, vr));
  rem = iadd(rem, imul(pv, ur));
  rem = iadd(rem, imul(ur, vr));
  put_scalars(r, uc * vc, uc * vat + vc * uat, rem, s1, s2);
}

// a + b / a - b (taylor_model.hpp:245-269); r may alias a or b.
template <bool SUB>
__device__ __forceinline__ void tm_addsub(Row& r, const Row& a, const Row& b, const Lane& L) {
  const double c = SUB ? a.c - b.c : a.c + b.c;
  const double at = SUB ? a.at - b.at : a.at + b.at;
  const Iv rem = SUB ? isub(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi}) : iadd(Iv{a.rlo, a.rhi}, Iv{b.rlo, b.rhi});
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    const double ra = SUB ? a.az[j] - b.az[j] : a.az[j] + b.az[j];
    const double rb = SUB ? a.bz[j] - b.bz[j] : a.bz[j] + b.bz[j];
    r.az[j] = ra;
    r.bz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  put_scalars(r, c, at, rem, s1, s2);
}

// s * a (+ d): scalar product (taylor_model.hpp:284-295) then + d (:302-306).
__device__ __forceinline__ void tm_affine(Row& r, double s, const Row& a, double d, const Lane& L) {
  const double c = a.c * s + d;
  const double at = a.at * s;
  const Iv rem = iscale(s, Iv{a.rlo, a.rhi});
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    const double ra = a.az[j] * s, rb = a.bz[j] * s;
    r.az[j] = ra;
    r.bz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  put_scalars(r, c, at, rem, s1, s2);
}

// sin / cos by linearization about the centre (taylor_model.hpp:397-425):
// r = f'(m) (u - m) + f(m) (+) [-rad^2/2, rad^2/2].  r may alias u.
template <bool COS>
__device__ __forceinline__ void tm_trig(Row& r, const Row& u, const Lane& L) {
  const double m = u.c;
  const Iv range = total_range(u, L.h);
  const double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
  const double err = rad * rad * 0.5;
  double sm, cm;
  sincos(m, &sm, &cm);
  const double s = COS ? -sm : cm;
  const double c = (m - m) * s + (COS ? cm : sm);  // (u - m) has centre u.c - m
  const double at = u.at * s;
  Iv rem = iscale(s, Iv{u.rlo, u.rhi});
  rem = iadd(rem, Iv{-err, err});
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < NZC; ++k) {
    if (!L.act[k]) continue;
    const int j = L.lane + 32 * k;
    const double ra = u.az[j] * s, rb = u.bz[j] * s;
    r.az[j] = ra;
    r.bz[j] = rb;
    s1 += fabs(ra);
    s2 += fabs(rb);
  }
  wsum2(s1, s2);
  put_scalars(r, c, at, rem, s1, s2);
}

// tme_inv (taylor_model.hpp:364-380); `thrown` replaces the domain_error.
__device__ __forceinline__ void tm_inv(Row& r, const Row& v, bool& thrown, const Lane& L) {
  const Iv range = total_range(v, L.h);
  if (range.lo <= 0.0 && range.hi >= 0.0) thrown = true;
  const double m = v.c;
  const double mm = m * m;
  const double e_lo = 1.0 / range.lo - (2.0 / m - range.lo / mm);
  const double e_hi = 1.0 / range.hi - (2.0 / m - range.hi / mm);
  const Iv e{smin(smin(e_lo, e_hi), 0.0), smax(smax(e_lo, e_hi), 0.0)};
  const double s = -1.0 / mm;
  tm_affine(r, s, v, 2.0 / m, L);
  r.rlo = r.rlo + e.lo;
  r.rhi = r.rhi + e.hi;
}

// ---------------------------------------------------------------------------
// make_augmented_field(12, 4, quadrotor_ode) (fields.hpp:96-107,
// systems.hpp:24-64) on the rows P[0..16) with temporaries T[0..NT).  Each
// derivative row dx_i is handed to consume(i, row) as soon as it exists
// (consume(i, nullptr) for the udot = 0 rows), in an order that lets a
// consumer overwrite P[i] (poly_picard's in-place update): P[i] is never
// read after dx_i is consumed.  The expression trees are the reference's,
// operand order included (TMExpr products are not commutative in rounding).
template <class Consume>
__device__ __forceinline__ bool quad_field(Row* P, Row* T, const double* prm, const Lane& L, Consume&& consume) {
  bool thrown = false;
  const double mass = prm[0], grav = prm[1], jx = prm[2], jy = prm[3], jz = prm[4];
  Row &sphi = T[0], &cphi = T[1], &sth = T[2], &cth = T[3], &spsi = T[4], &cpsi = T[5];
  Row &a = T[6], &t1 = T[7], &t2 = T[8], &t3 = T[9];
  const Row &p = P[9], &q = P[10], &r = P[11];
  consume(0, &P[3]);
  consume(1, &P[4]);
  consume(2, &P[5]);
  tm_trig<false>(sphi, P[6], L);
  tm_trig<true>(cphi, P[6], L);
  tm_trig<false>(sth, P[7], L);
  tm_trig<true>(cth, P[7], L);
  tm_trig<false>(spsi, P[8], L);
  tm_trig<true>(cpsi, P[8], L);
  tm_affine(a, 1.0 / mass, P[12], 0.0, L);
  // b3x = cphi*sth*cpsi + sphi*spsi ; dx3 = a*b3x
  tm_mul(t1, cphi, sth, L);
  tm_mul(t2, t1, cpsi, L);
  tm_mul(t3, sphi, spsi, L);
  tm_addsub<false>(t2, t2, t3, L);
  tm_mul(t3, a, t2, L);
  consume(3, &t3);
  // b3y = cphi*sth*spsi - sphi*cpsi ; dx4 = a*b3y
  tm_mul(t2, t1, spsi, L);
  tm_mul(t3, sphi, cpsi, L);
  tm_addsub<true>(t2, t2, t3, L);
  tm_mul(t3, a, t2, L);
  consume(4, &t3);
  // dx5 = a*(cphi*cth) - g
  tm_mul(t2, cphi, cth, L);
  tm_mul(t3, a, t2, L);
  t3.c = t3.c - grav;
  consume(5, &t3);
  // tth = sth / cth = sth * tme_inv(cth); `a` now holds tme_inv(cth)
  tm_inv(a, cth, thrown, L);
  tm_mul(t1, sth, a, L);
  // dx6 = p + sphi*tth*q + cphi*tth*r
  tm_mul(t2, sphi, t1, L);
  tm_mul(t2, t2, q, L);
  tm_addsub<false>(t2, p, t2, L);
  tm_mul(t3, cphi, t1, L);
  tm_mul(t3, t3, r, L);
  tm_addsub<false>(t3, t2, t3, L);
  consume(6, &t3);
  // dx7 = cphi*q - sphi*r
  tm_mul(t2, cphi, q, L);
  tm_mul(t3, sphi, r, L);
  tm_addsub<true>(t2, t2, t3, L);
  consume(7, &t2);
  // dx8 = (sphi/cth)*q + (cphi/cth)*r (each division re-evaluates tme_inv(cth): same value)
  tm_mul(t2, sphi, a, L);
  tm_mul(t2, t2, q, L);
  tm_mul(t3, cphi, a, L);
  tm_mul(t3, t3, r, L);
  tm_addsub<false>(t2, t2, t3, L);
  consume(8, &t2);
  // dx9..11 = (rate products) * inertia ratio + torque / inertia
  tm_mul(T[0], q, r, L);
  tm_affine(T[0], (jy - jz) / jx, T[0], 0.0, L);
  tm_affine(T[1], 1.0 / jx, P[13], 0.0, L);
  tm_addsub<false>(T[0], T[0], T[1], L);
  tm_mul(T[1], p, r, L);
  tm_affine(T[1], (jz - jx) / jy, T[1], 0.0, L);
  tm_affine(T[2], 1.0 / jy, P[14], 0.0, L);
  tm_addsub<false>(T[1], T[1], T[2], L);
  tm_mul(T[2], p, q, L);
  tm_affine(T[2], (jx - jy) / jz, T[2], 0.0, L);
  tm_affine(T[3], 1.0 / jz, P[15], 0.0, L);
  tm_addsub<false>(T[2], T[2], T[3], L);
  consume(9, &T[0]);
  consume(10, &T[1]);
  consume(11, &T[2]);
#pragma unroll
  for (int i = 12; i < NA; ++i) consume(i, static_cast<const Row*>(nullptr));
  return thrown;
}

// ---------------------------------------------------------------------------
// Shared memory of one flow warp.
struct FlowSmem {
  Row P[NA];          // the Picard iterate p_k (candidate remainders in rem)
  Row T[NT];          // field temporaries
  double S[NA * LDS];  // seed / endpoint generator rows [G0 | Q1..Qnq], stride LDS
  double sc[NA];      // seed centre
  double ssz[NA];     // abs_z of the seed rows
  double ec[NA];      // endpoint centre
  Iv erem[NA];        // endpoint remainder
  Iv i0[NA], i1[NA], nx[NA];
};

__device__ __forceinline__ void emit_box(const CTParams& P, long long b, int k, int d, double lo, double hi) {
  if (!P.split) {
    const size_t o = (static_cast<size_t>(b) * P.T + k) * NA + d;
    P.out_lo[o] = lo;
    P.out_hi[o] = hi;
  } else {
    if (lo == lo) atomicMin(&P.hull_lo[k * NA + d], order_key(lo));
    if (hi == hi) atomicMax(&P.hull_hi[k * NA + d], order_key(hi));
    if (P.part_begin + b == 0) {
      if (lo != lo) P.hull_nan0[(k * NA + d) * 2 + 0] = 1;
      if (hi != hi) P.hull_nan0[(k * NA + d) * 2 + 1] = 1;
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

// hull fold of fold_overflow (flowpipe_ct.hpp:347-348) on the shared state:
// the oldest block (columns [p0, p0 + NA)) is boxed into the newest block's
// diagonal (columns [nz - NA, nz)), then dropped.  Lane i < NA sweeps row i
// sequentially (the reference's row_abs_sum order).
__device__ __forceinline__ void fold_hull(double* S, int p0, int& nz, int& nq, int cap, int lane) {
  while (nq > cap) {
    __syncwarp();
    if (lane < NA) {
      double r = 0.0;
      for (int j = 0; j < NA; ++j) r += fabs(S[lane * LDS + p0 + j]);
      S[lane * LDS + (nz - NA) + lane] += r;
    }
    __syncwarp();
    for (int i = 0; i < NA; ++i) {
      double v[NZC];
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        v[k] = (j >= p0 && j + NA < nz) ? S[i * LDS + j + NA] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (j >= p0 && j < nz) S[i * LDS + j] = v[k];
      }
    }
    __syncwarp();
    nz -= NA;
    nq -= 1;
  }
}

// ---------------------------------------------------------------------------
// k_atomic flowpipe steps of one control interval, one warp per sub-box.
__global__ void __launch_bounds__(32) ct_flow_kernel(const CTParams Pm) {
  extern __shared__ __align__(16) unsigned char ct_smem[];
  FlowSmem& W = *reinterpret_cast<FlowSmem*>(ct_smem);
  const long long b = blockIdx.x;
  if (b >= Pm.B) return;
  const int lane = threadIdx.x;
  int* meta = Pm.st_meta + b * 4;
  int nq = meta[0], status = meta[1], fstep = meta[2], nboxes = meta[3];
  const bool last = (Pm.ci + 1 == Pm.ctl_steps);
  if (status != CT_OK) {
    if (last && lane == 0) finalize(Pm, b, nboxes, status, fstep);
    return;
  }
  const double h = Pm.h;
  const int p0 = Pm.n;
  const int cap = Pm.window > 0 ? Pm.window : 1;
  int nz = p0 + nq * NA;
  // load the state; zero every row's padding once (ops never write it)
  {
    const double* gM = Pm.st_M + static_cast<size_t>(b) * NA * NZP;
    for (int i = 0; i < NA; ++i) {
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        W.S[i * LDS + j] = gM[i * NZP + j];
        W.P[i].az[j] = 0.0;
        W.P[i].bz[j] = 0.0;
      }
    }
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        W.T[t].az[lane + 32 * k] = 0.0;
        W.T[t].bz[lane + 32 * k] = 0.0;
      }
    if (lane < NA) W.sc[lane] = Pm.st_c[b * NA + lane];
  }
  __syncwarp();

  Lane L;
  L.lane = lane;
  L.h = h;
  for (int step = 0; step < Pm.K && status == CT_OK; ++step) {
    const int gstep = Pm.ci * Pm.K + step;
#pragma unroll
    for (int k = 0; k < NZC; ++k) L.act[k] = (lane + 32 * k) < nz;
    // seed rows: abs_z of each (cached for the Picard rows)
    for (int i = 0; i < NA; i += 2) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        if (!L.act[k]) continue;
        const int j = lane + 32 * k;
        s1 += fabs(W.S[i * LDS + j]);
        s2 += fabs(W.S[(i + 1) * LDS + j]);
      }
      wsum2(s1, s2);
      W.ssz[i] = s1;
      W.ssz[i + 1] = s2;
    }
    // poly_picard (flowpipe_ct.hpp:126-139): g_0 = seed
    for (int i = 0; i < NA; ++i) {
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        if (!L.act[k]) continue;
        const int j = lane + 32 * k;
        W.P[i].az[j] = W.S[i * LDS + j];
        W.P[i].bz[j] = 0.0;
      }
      put_scalars(W.P[i], W.sc[i], 0.0, Iv{0.0, 0.0}, W.ssz[i], 0.0);
    }
    // g_{j+1} = seed + Int f(g_j), rows overwritten in place as dx_i appears
    auto picard = [&](int i, const Row* f) {
      Row& g = W.P[i];
      const double fc = f ? f->c : 0.0, fat = f ? f->at : 0.0, fsz = f ? f->sz : 0.0, fsb = f ? f->sb : 0.0;
      const Iv fr = f ? Iv{f->rlo, f->rhi} : Iv{0.0, 0.0};
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        if (!L.act[k]) continue;
        const int j = lane + 32 * k;
        const double fa = f ? f->az[j] : 0.0;
        g.az[j] = W.S[i * LDS + j];
        g.bz[j] = fa;
      }
      // tme_integrate (taylor_model.hpp:429-445) rem, added to the seed's [0, 0]
      const double half_at = fat * 0.5;
      Iv rem = imul(Iv{0.0, h * h}, Iv{half_at, half_at});
      const double bb = fsb * h * h * 0.5;
      rem = iadd(rem, Iv{-bb, bb});
      rem = iadd(rem, imul(fr, Iv{0.0, h}));
      put_scalars(g, W.sc[i], fc, rem, W.ssz[i], fsz);
    };
    bool thrown = false;
    for (int it = 0; it < Pm.order && !thrown; ++it) thrown = quad_field(W.P, W.T, Pm.prm, L, picard);
    int fail = CT_OK;
    if (thrown) fail = CT_TME_INV;
    if (fail == CT_OK) {
      for (int i = 0; i < NA; ++i)
        if (!isfinite(W.P[i].c)) fail = CT_PICARD;
    }
    // remainder_picard (flowpipe_ct.hpp:144-276)
    auto replay = [&](const Iv* cand) {  // I1 induced by candidate remainder `cand` (:154-165)
      for (int i = 0; i < NA; ++i) {
        W.P[i].rlo = cand[i].lo;
        W.P[i].rhi = cand[i].hi;
      }
      auto induced = [&](int i, const Row* f) {
        const Row& pk = W.P[i];
        const double fc = f ? f->c : 0.0, fat = f ? f->at : 0.0, fsb = f ? f->sb : 0.0;
        const Iv fr = f ? Iv{f->rlo, f->rhi} : Iv{0.0, 0.0};
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int k = 0; k < NZC; ++k) {
          if (!L.act[k]) continue;
          const int j = lane + 32 * k;
          const double fa = f ? f->az[j] : 0.0;
          s1 += fabs(W.S[i * LDS + j] - pk.az[j]);
          s2 += fabs(fa - pk.bz[j]);
        }
        wsum2(s1, s2);
        // (seed + Int f) - p_k with p_k's own remainder [0, 0]
        const double half_at = fat * 0.5;
        Iv rem = imul(Iv{0.0, h * h}, Iv{half_at, half_at});
        const double bb = fsb * h * h * 0.5;
        rem = iadd(rem, Iv{-bb, bb});
        rem = iadd(rem, imul(fr, Iv{0.0, h}));
        const double dc = W.sc[i] - pk.c, dat = fc - pk.at;
        const Iv r = iadd(poly_range(dc, s1, dat, s2, h), rem);
        W.nx[i] = r;
      };
      return quad_field(W.P, W.T, Pm.prm, L, induced);
    };
    auto finite_box = [&](const Iv* x) {
      bool ok = true;
      for (int i = 0; i < NA; ++i) ok = ok && ifin(x[i]);
      return ok;
    };
    auto subset = [&](const Iv* in, const Iv* out) {
      bool ok = true;
      for (int i = 0; i < NA; ++i) ok = ok && (out[i].lo <= in[i].lo && in[i].hi <= out[i].hi);
      return ok;
    };
    if (fail == CT_OK) {
      for (int i = 0; i < NA; ++i) {
        W.P[i].rlo = 0.0;
        W.P[i].rhi = 0.0;
        W.i0[i] = Iv{-Pm.eps, Pm.eps};
        W.i1[i] = Iv{0.0, 0.0};
      }
      bool accepted = false;
      for (int attempt = 0; attempt <= Pm.maxe; ++attempt) {
        const bool threw = replay(W.i0);
        if (!threw)
          for (int i = 0; i < NA; ++i) W.i1[i] = W.nx[i];
        if (!threw && finite_box(W.i1) && subset(W.i1, W.i0)) {
          accepted = true;
          break;
        }
        for (int i = 0; i < NA; ++i) {  // per-dimension adaptive enlargement (:178-182)
          const Iv ind = threw ? Iv{0.0, 0.0} : W.i1[i];
          const Iv cur = W.i0[i];
          const Iv hull = (ind.lo <= ind.hi) ? Iv{smin(cur.lo, ind.lo), smax(cur.hi, ind.hi)} : cur;
          const double mid = (hull.lo + hull.hi) * 0.5, rad = (hull.hi - hull.lo) * 0.5 * Pm.enl;
          W.i0[i] = Iv{mid - rad, mid + rad};
        }
      }
      if (!accepted) fail = CT_REMAINDER;
    }
    if (fail == CT_OK) {
      for (int round = 0; round < Pm.refine; ++round) {  // shrink (:214-223)
        if (replay(W.i1)) break;
        if (!(finite_box(W.nx) && subset(W.nx, W.i1))) break;
        for (int i = 0; i < NA; ++i) W.i1[i] = W.nx[i];
      }
      // endpoint by exact integration at tau = h (:236-263), written over the seed rows
      for (int i = 0; i < NA; ++i) {
        W.P[i].rlo = W.i1[i].lo;
        W.P[i].rhi = W.i1[i].hi;
      }
      auto endpoint = [&](int i, const Row* f) {
        const double fc = f ? f->c : 0.0, fat = f ? f->at : 0.0;
        const Iv fr = f ? Iv{f->rlo, f->rhi} : Iv{0.0, 0.0};
#pragma unroll
        for (int k = 0; k < NZC; ++k) {
          if (!L.act[k]) continue;
          const int j = lane + 32 * k;
          const double fa = f ? f->az[j] : 0.0, fb = f ? f->bz[j] : 0.0;
          W.S[i * LDS + j] = W.S[i * LDS + j] + h * (fa + fb * h * 0.5);
        }
        W.ec[i] = W.sc[i] + h * (fc + fat * h * 0.5);
        W.erem[i] = iadd(imul(Iv{h, h}, fr), Iv{0.0, 0.0});
      };
      const bool threw = quad_field(W.P, W.T, Pm.prm, L, endpoint);
      bool exact_ok = !threw && finite_box(W.erem);
      for (int i = 0; i < NA; ++i) exact_ok = exact_ok && isfinite(W.ec[i]);
      if (!exact_ok) {  // fallback: the certified segment at tau = h (:264-274)
        for (int i = 0; i < NA; ++i) {
#pragma unroll
          for (int k = 0; k < NZC; ++k) {
            if (!L.act[k]) continue;
            const int j = lane + 32 * k;
            W.S[i * LDS + j] = W.P[i].az[j] + W.P[i].bz[j] * h;
          }
          W.ec[i] = W.P[i].c + W.P[i].at * h;
          W.erem[i] = W.i1[i];
        }
      }
      // tm_eval_interval(segment, [0, h]) (taylor_model.hpp:73-97)
      bool fin = true;
      const int kbox = 1 + gstep;
      double blo = 0.0, bhi = 0.0;
      for (int i = 0; i < NA; ++i) {
        const Row& p = W.P[i];
        Iv acc{p.c - p.sz, p.c + p.sz};
        acc = iadd(acc, iscale(p.at, Iv{0.0, h}));
        const double tau_mag = smax(0.0, h);
        acc = iadd(acc, Iv{-p.sb * tau_mag, p.sb * tau_mag});
        acc = iadd(acc, W.i1[i]);
        fin = fin && ifin(acc);
        if (lane == i) {
          blo = acc.lo;
          bhi = acc.hi;
        }
      }
      if (lane < NA) emit_box(Pm, b, kbox, lane, blo, bhi);
      nboxes = kbox + 1;
      if (!fin) {
        fail = CT_BOX;
      } else {
        // symbolic_step (flowpipe_ct.hpp:378-409): centre the remainder, push
        // its radius as a fresh diagonal block, fold the overflow
        __syncwarp();
        for (int i = 0; i < NA; ++i) {
#pragma unroll
          for (int k = 0; k < NZC; ++k) {
            const int j = lane + 32 * k;
            if (j >= nz && j < nz + NA)
              W.S[i * LDS + j] = (j - nz == i) ? (W.erem[i].hi - W.erem[i].lo) * 0.5 : 0.0;
          }
        }
        if (lane < NA) W.sc[lane] = W.ec[lane] + (W.erem[lane].lo + W.erem[lane].hi) * 0.5;
        nz += NA;
        nq += 1;
        fold_hull(W.S, p0, nz, nq, cap, lane);
      }
    }
    if (fail != CT_OK) {
      status = fail;
      fstep = gstep;
    }
  }
  // write the state back
  __syncwarp();
  {
    double* gM = Pm.st_M + static_cast<size_t>(b) * NA * NZP;
    for (int i = 0; i < NA; ++i)
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        gM[i * NZP + j] = (j < nz) ? W.S[i * LDS + j] : 0.0;
      }
    if (lane < NA) Pm.st_c[b * NA + lane] = W.sc[lane];
  }
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
struct CtlSmem {
  double xA[NX * LDX];           // state TM rows (n x nzx), stride LDX
  double xc[NX];
  double pre[kMaxLayers][kMaxCtlW][2];  // preactivation boxes of the hidden layers
  double hb[2][kMaxCtlW][2];     // IBP boxes
  double lam[2][4][NZP + 32];    // Lambda (n_o x width), double buffered
  double bf0[kMaxCtlW];          // frozen first-layer bias
  double blo[4], bup[4];
  double uc[4];
  Iv urem[4];
};

constexpr int kCtlWarps = 4;

__device__ __forceinline__ void relax_tanh_or_relu(int act, double l, double u, double& s, double& li, double& ui) {
  relax(act, l, u, s, li, ui);
}

__global__ void __launch_bounds__(32 * kCtlWarps) ct_ctl_kernel(const CTParams Pm) {
  extern __shared__ __align__(16) unsigned char ct_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  CtlSmem& W = reinterpret_cast<CtlSmem*>(ct_smem)[warp];
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
    for (int i = 0; i < n; ++i)
      for (int j = lane; j < nzx; j += 32) W.xA[i * LDX + j] = gM[i * NZP + j];
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
      for (int j = 0; j < in_cols; ++j) {
        const double w = blob[N.wt_off[t] + static_cast<size_t>(j) * N.ldt[t] + u];
        const double xl = W.hb[cur][j][0], xh = W.hb[cur][j][1];
        lo = lo + ((w >= 0.0) ? w * xl : w * xh);
        hi = hi + ((w >= 0.0) ? w * xh : w * xl);
      }
      const double bias = (t == 0) ? W.bf0[u] : blob[N.b_off[t] + u];
      lo = lo + bias;
      hi = hi + bias;
      W.pre[t][u][0] = lo;
      W.pre[t][u][1] = hi;
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
      const double pl = W.pre[t][u][0], ph = W.pre[t][u][1];
      if (!(isfinite(pl) && isfinite(ph))) {
        bad = true;
        s = li = ui = 0.0;
      } else {
        relax(N.acts[t], pl, ph, s, li, ui);
      }
      W.pre[t][u][0] = s;
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
        W.lam[lb][lane][j] = aij * W.pre[t][j][0];
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
      for (int k = 0; k < width; ++k) {
        const double w = blob[N.w_off[t] + static_cast<size_t>(k) * N.ldw[t] + jc];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < no) acc[i] = acc[i] + W.lam[lb][i][k] * w;
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
      if (i < no) S[i * (NZP + 32) + jc] = acc[i];
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
  // ---- stacking (closed_loop.hpp:122-153) into global memory
  int nz = nzx + NA;
  int nqn = nbw + 1;
  for (int d = 0; d < NA; ++d) {
    for (int j = lane; j < NZP; j += 32) {
      double v = 0.0;
      if (j < nzx) {
        v = (d < n) ? W.xA[d * LDX + j] : S[(d - n) * (NZP + 32) + j];
      } else if (j - nzx == d) {
        v = (d < n) ? (0.0 - 0.0) * 0.5 : (W.urem[d - n].hi - W.urem[d - n].lo) * 0.5;
      }
      gM[d * NZP + j] = v;
    }
  }
  if (lane < NA) gc[lane] = (lane < n) ? W.xc[lane] + (0.0 + 0.0) * 0.5
                                       : W.uc[lane - n] + (W.urem[lane - n].lo + W.urem[lane - n].hi) * 0.5;
  __syncwarp();
  __threadfence_block();
  // fold_overflow hull branch (flowpipe_ct.hpp:347-348), G0 = (n + l) x n is never square
  while (nqn > cap) {
    if (lane < NA) {
      double r = 0.0;
      for (int j = 0; j < NA; ++j) r += fabs(gM[lane * NZP + n + j]);
      gM[lane * NZP + (nz - NA) + lane] += r;
    }
    __syncwarp();
    __threadfence_block();
    for (int d = 0; d < NA; ++d) {
      double v[NZC];
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        v[k] = (j >= n && j + NA < nz) ? gM[d * NZP + j + NA] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < NZC; ++k) {
        const int j = lane + 32 * k;
        if (j >= n && j < nz) gM[d * NZP + j] = v[k];
      }
      __syncwarp();
    }
    __threadfence_block();
    nz -= NA;
    nqn -= 1;
  }
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
      emit_box(Pm, b, 0, lane, c - r, c + r);
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
