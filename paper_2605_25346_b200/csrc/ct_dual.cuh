// Forward-mode (reach::Dual) tangents through the continuous-time closed loop: the gradient of
// ctl_reach_loss (training.hpp:183-213) over the controller's parameters, as grad_forward
// (refine.hpp:186-207) evaluates it -- one Dual pass of cl_reach (closed_loop.hpp:76-182) per seeded
// parameter and episode.
//
// One warp per (pass p, episode e); its working set (~200 KB) in global memory (L1 / L2 resident) with 12
// persistent passes per SM (ctl_reach_loss_grad_kernel_g, the default: 3.6x the one-pass-per-SM
// shared-memory variant ctl_reach_loss_grad_kernel, RB_CTD_SLOTS_PER_SM=0; swept 8 / 10 / 12 / 14 / 16 / 24):
//   * TMExpr<Dual> rows (taylor_model.hpp:197-445) with the generator columns lane-strided
//     (lane L owns columns L, L+32, L+64); the scalar parts (c, at, the remainder interval) are
//     computed by every lane alike and stored by lane 0; abs-sums are warp reductions;
//   * the quadrotor field under make_augmented_field (systems.hpp:24-64, fields.hpp:96-128),
//     poly_picard / remainder_picard (flowpipe_ct.hpp:126-276), tm_eval_interval, symbolic_step and
//     the box-hull fold_overflow (flowpipe_ct.hpp:317-424; G0 is (n+l) x n in cl_reach, never square);
//   * ctl_crown (neural.hpp:398-424): the reference folded into the first-layer bias, certify_tm_input
//     with the tanh / ReLU relaxations (relax_d) in Dual, the network read through a NetView whose
//     one seeded entry carries the tangent.
// Every branch reads primal values only (reach's rule), so the primal part of each pass is the
// primal cl_reach; the per-episode term log(1 + predicted_volume) (or the cap) goes to the host.
// The abs-sums are tree reductions and sin / cos / tanh are CUDA's: values agree with the reference
// to ~1e-15 relative, tangents within 1e-9 (tests/test_gpu_ctl_grad.py).
#pragma once

#include "dual_kernel.cuh"

namespace rb {
namespace ctd {

using dual::D;
using dual::DI;
using dual::dabs;
using dual::dadd;
using dual::dc;
using dual::dcos;
using dual::ddiv;
using dual::dfin;
using dual::dmax;
using dual::dmin;
using dual::dmul;
using dual::dneg;
using dual::dsin;
using dual::dsub;
using dual::iadd;    // interval.hpp:60-62 on Interval<Dual>
using dual::imid;
using dual::irad;
using dual::iscale;  // interval.hpp:80-84

#ifndef RB_CTD_MIN_BLOCKS
#define RB_CTD_MIN_BLOCKS 12  // passes per SM the global-memory variant is compiled for (<= 170 registers)
#endif
constexpr int MZ = 96;  // generator columns (n + l + window * (n + l) <= 96)
constexpr int MR = 16;  // rows of the augmented state (n + l)
constexpr int CW = 128; // widest controller layer
constexpr int CO = 8;   // controller outputs (l)
constexpr int CA = 128; // Lambda row length (>= widest layer and nz + n)

struct TM {
  D c, at;
  DI rem;
  D az[MZ];
  D bz[MZ];
};

// interval.hpp:60-94 on Interval<Dual> (outward rounding off)
__device__ __forceinline__ DI isub(DI a, DI b) { return DI{dsub(a.lo, b.hi), dsub(a.hi, b.lo)}; }
__device__ __forceinline__ DI imul(DI a, DI b) {
  const D p1 = dmul(a.lo, b.lo), p2 = dmul(a.lo, b.hi), p3 = dmul(a.hi, b.lo), p4 = dmul(a.hi, b.hi);
  return DI{dmin(dmin(p1, p2), dmin(p3, p4)), dmax(dmax(p1, p2), dmax(p3, p4))};
}
__device__ __forceinline__ DI ihull(DI a, DI b) { return DI{dmin(a.lo, b.lo), dmax(a.hi, b.hi)}; }
__device__ __forceinline__ DI ipt(D v) { return DI{v, v}; }
__device__ __forceinline__ DI izero() { return DI{dc(0.0), dc(0.0)}; }
__device__ __forceinline__ bool ifin(DI x) { return isfinite(x.lo.v) && isfinite(x.hi.v); }
__device__ __forceinline__ bool ivalid(DI x) { return x.lo.v <= x.hi.v; }
__device__ __forceinline__ bool isubset(DI in, DI out) { return out.lo.v <= in.lo.v && in.hi.v <= out.hi.v; }

__device__ __forceinline__ D wsum(D v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v.v = add(v.v, __shfl_xor_sync(0xffffffffu, v.v, o));
    v.d = add(v.d, __shfl_xor_sync(0xffffffffu, v.d, o));
  }
  return v;
}
// sum_j abs(x[j]) over nz lane-strided columns (reach::abs on Dual)
__device__ __forceinline__ D abs_sum(const D* x, int nz) {
  const int lane = threadIdx.x & 31;
  D a = dc(0.0);
  for (int j = lane; j < nz; j += 32) a = dadd(a, dabs(x[j]));
  return wsum(a);
}

// Scalar part of a TM row, read by every lane.
struct Sc {
  D c, at;
  DI rem;
};
__device__ __forceinline__ Sc ld(const TM* t) { return Sc{t->c, t->at, t->rem}; }
__device__ __forceinline__ void st(TM* t, const Sc& s) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    t->c = s.c;
    t->at = s.at;
    t->rem = s.rem;
  }
  __syncwarp();
}

// poly_range (taylor_model.hpp:227-235) given the abs-sums
__device__ __forceinline__ DI poly_range(const Sc& u, D zr, D br0, double h) {
  DI r{dsub(u.c, zr), dadd(u.c, zr)};
  r = iadd(r, imul(DI{dc(0.0), dc(h)}, DI{u.at, u.at}));
  const D br = dmul(br0, dc(h));
  return iadd(r, DI{dneg(br), br});
}

__device__ __forceinline__ void tm_const(TM* r, D v, int nz) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dc(0.0);
    r->bz[j] = dc(0.0);
  }
  st(r, Sc{v, dc(0.0), izero()});
}
__device__ __forceinline__ void tm_copy(TM* r, const TM* a, int nz) {
  const int lane = threadIdx.x & 31;
  const Sc s = ld(a);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = a->az[j];
    r->bz[j] = a->bz[j];
  }
  st(r, s);
}
// operator+ / operator- (taylor_model.hpp:245-269); r may alias a or b
__device__ __forceinline__ void tm_add(TM* r, const TM* a, const TM* b, int nz) {
  const int lane = threadIdx.x & 31;
  const Sc x = ld(a), y = ld(b);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dadd(a->az[j], b->az[j]);
    r->bz[j] = dadd(a->bz[j], b->bz[j]);
  }
  st(r, Sc{dadd(x.c, y.c), dadd(x.at, y.at), iadd(x.rem, y.rem)});
}
__device__ __forceinline__ void tm_sub(TM* r, const TM* a, const TM* b, int nz) {
  const int lane = threadIdx.x & 31;
  const Sc x = ld(a), y = ld(b);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dsub(a->az[j], b->az[j]);
    r->bz[j] = dsub(a->bz[j], b->bz[j]);
  }
  st(r, Sc{dsub(x.c, y.c), dsub(x.at, y.at), isub(x.rem, y.rem)});
}
// s * TM (taylor_model.hpp:284-295): r.x *= s, rem = iv_scale(s, a.rem); r may alias a
__device__ __forceinline__ void tm_smul(TM* r, D s, const TM* a, int nz) {
  const int lane = threadIdx.x & 31;
  const Sc x = ld(a);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dmul(a->az[j], s);
    r->bz[j] = dmul(a->bz[j], s);
  }
  st(r, Sc{dmul(x.c, s), dmul(x.at, s), iscale(s, x.rem)});
}
// TM + s / TM - s (taylor_model.hpp:302-317); in place
__device__ __forceinline__ void tm_sadd(TM* r, D s) {
  Sc x = ld(r);
  x.c = dadd(x.c, s);
  st(r, x);
}
__device__ __forceinline__ void tm_ssub(TM* r, D s) {
  Sc x = ld(r);
  x.c = dsub(x.c, s);
  st(r, x);
}

// operator* (taylor_model.hpp:325-360); r must not alias u or v
__device__ __forceinline__ void tm_mul(TM* r, const TM* u, const TM* v, int nz, double hd) {
  const int lane = threadIdx.x & 31;
  const Sc U = ld(u), V = ld(v);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dadd(dmul(U.c, v->az[j]), dmul(V.c, u->az[j]));
    r->bz[j] = dadd(dadd(dadd(dmul(U.c, v->bz[j]), dmul(V.c, u->bz[j])), dmul(U.at, v->az[j])), dmul(V.at, u->az[j]));
  }
  const D h = dc(hd);
  const D au = abs_sum(u->az, nz), av = abs_sum(v->az, nz), bu = abs_sum(u->bz, nz), bv = abs_sum(v->bz, nz);
  const D atu = dabs(U.at), atv = dabs(V.at);
  D sym = dmul(au, av);
  sym = dadd(sym, dmul(dadd(dmul(au, bv), dmul(av, bu)), h));
  sym = dadd(sym, dmul(dmul(dmul(bu, bv), h), h));
  sym = dadd(sym, dmul(dmul(dadd(dmul(atu, bv), dmul(atv, bu)), h), h));
  DI rem = izero();
  rem = iadd(rem, DI{dneg(sym), sym});
  const D tt = dmul(U.at, V.at);
  rem = iadd(rem, imul(DI{dc(0.0), dmul(h, h)}, DI{tt, tt}));
  const DI pu = poly_range(U, au, bu, hd), pv = poly_range(V, av, bv, hd);
  rem = iadd(rem, imul(pu, V.rem));
  rem = iadd(rem, imul(pv, U.rem));
  rem = iadd(rem, imul(U.rem, V.rem));
  st(r, Sc{dmul(U.c, V.c), dadd(dmul(U.c, V.at), dmul(V.c, U.at)), rem});
}

// total_range (taylor_model.hpp:237)
__device__ __forceinline__ DI total_range(const TM* u, int nz, double h) {
  const Sc U = ld(u);
  return iadd(poly_range(U, abs_sum(u->az, nz), abs_sum(u->bz, nz), h), U.rem);
}

// tme_inv (taylor_model.hpp:364-380); sets thrown on a zero-containing range (r may not alias v)
__device__ __forceinline__ void tm_inv(TM* r, const TM* v, int nz, double h, bool& thrown) {
  const DI range = total_range(v, nz, h);
  if (range.lo.v <= 0.0 && range.hi.v >= 0.0) thrown = true;
  const D m = ld(v).c;
  const D mm = dmul(m, m);
  auto err = [&](D x) { return dsub(ddiv(dc(1.0), x), dsub(ddiv(dc(2.0), m), ddiv(x, mm))); };
  const D e_lo = err(range.lo), e_hi = err(range.hi);
  const DI e{dmin(dmin(e_lo, e_hi), dc(0.0)), dmax(dmax(e_lo, e_hi), dc(0.0))};
  tm_smul(r, ddiv(dc(-1.0), mm), v, nz);
  tm_sadd(r, ddiv(dc(2.0), m));
  Sc x = ld(r);
  x.rem = iadd(x.rem, e);
  st(r, x);
}

// sin / cos (taylor_model.hpp:397-425); r must not alias u
__device__ __forceinline__ void tm_sincos(TM* r, const TM* u, int nz, double h, bool is_cos) {
  const D m = ld(u).c;
  const DI range = total_range(u, nz, h);
  const D rad = dmax(dabs(dsub(range.lo, m)), dabs(dsub(range.hi, m)));
  const D err = dmul(dmul(rad, rad), dc(0.5));
  tm_copy(r, u, nz);
  tm_ssub(r, m);
  tm_smul(r, is_cos ? dneg(dsin(m)) : dcos(m), r, nz);
  tm_sadd(r, is_cos ? dcos(m) : dsin(m));
  Sc x = ld(r);
  x.rem = iadd(x.rem, DI{dneg(err), err});
  st(r, x);
}

// tme_integrate (taylor_model.hpp:429-445); r must not alias u
__device__ __forceinline__ void tm_integrate(TM* r, const TM* u, int nz, double hd) {
  const int lane = threadIdx.x & 31;
  const Sc U = ld(u);
  for (int j = lane; j < nz; j += 32) {
    r->az[j] = dc(0.0);
    r->bz[j] = u->az[j];
  }
  const D h = dc(hd);
  DI rem = izero();
  const D half_at = dmul(U.at, dc(0.5));
  rem = iadd(rem, imul(DI{dc(0.0), dmul(h, h)}, DI{half_at, half_at}));
  const D bb = dmul(dmul(dmul(abs_sum(u->bz, nz), h), h), dc(0.5));
  rem = iadd(rem, DI{dneg(bb), bb});
  rem = iadd(rem, imul(U.rem, DI{dc(0.0), h}));
  st(r, Sc{dc(0.0), U.c, rem});
}

// Shared-memory working set of one pass.
struct Work {
  D sc[MR];
  D sM[MR][MZ];  // symbolic state [G0 | Q1 .. Qnq] (flowpipe_ct.hpp:286-300)
  int wid[16];
  int p0, nq;
  DI i0[MR], i1[MR], nx[MR], erem[MR];
  D ec[MR];
  TM g[MR];      // Picard iterate; after poly_picard the polynomial p_k (rem zeroed)
  TM t[14];      // quad_body temporaries, d1, d2
  union {
    TM fg[MR];   // field output
    struct {     // controller certification (not live during a flow step)
      DI pre[kMaxLayers][CW];
      DI hb[2][CW];
      D a[CO][CA];
      D an[CO][CA];
      D sl[CW], li[CW], ui[CW];
      D blo[CO], bup[CO], uc[CO];
      DI urem[CO];
      D b0[CW];  // frozen first-layer bias
      D xc[MR];
    } cc;
  };
};

// quadrotor_ode (systems.hpp:24-64) on TM rows x[0..12) with inputs u[0..4), as ct_oracle.c quad_body
__device__ void quad_body(const TM* x, const TM* u, TM* dx, const double* prm, TM* t, int nz, double h,
                          bool& thrown) {
  const double mass = prm[0], grav = prm[1], jx = prm[2], jy = prm[3], jz = prm[4];
  TM *sphi = &t[0], *cphi = &t[1], *sth = &t[2], *cth = &t[3], *spsi = &t[4], *cpsi = &t[5];
  TM *a = &t[6], *t1 = &t[7], *t2 = &t[8], *t3 = &t[9], *ic = &t[10], *tth = &t[11];
  const TM *phi = &x[6], *theta = &x[7], *psi = &x[8], *p = &x[9], *q = &x[10], *r = &x[11];
  tm_sincos(sphi, phi, nz, h, false);
  tm_sincos(cphi, phi, nz, h, true);
  tm_sincos(sth, theta, nz, h, false);
  tm_sincos(cth, theta, nz, h, true);
  tm_sincos(spsi, psi, nz, h, false);
  tm_sincos(cpsi, psi, nz, h, true);
  tm_smul(a, dc(1.0 / mass), &u[0], nz);
  tm_copy(&dx[0], &x[3], nz);
  tm_copy(&dx[1], &x[4], nz);
  tm_copy(&dx[2], &x[5], nz);
  tm_mul(t1, cphi, sth, nz, h);
  tm_mul(t2, t1, cpsi, nz, h);
  tm_mul(t3, sphi, spsi, nz, h);
  tm_add(t2, t2, t3, nz);
  tm_mul(&dx[3], a, t2, nz, h);
  tm_mul(t2, t1, spsi, nz, h);
  tm_mul(t3, sphi, cpsi, nz, h);
  tm_sub(t2, t2, t3, nz);
  tm_mul(&dx[4], a, t2, nz, h);
  tm_mul(t2, cphi, cth, nz, h);
  tm_mul(t3, a, t2, nz, h);
  tm_copy(&dx[5], t3, nz);
  tm_ssub(&dx[5], dc(grav));
  tm_inv(ic, cth, nz, h, thrown);
  tm_mul(tth, sth, ic, nz, h);
  tm_mul(t1, sphi, tth, nz, h);
  tm_mul(t2, t1, q, nz, h);
  tm_add(t2, p, t2, nz);
  tm_mul(t1, cphi, tth, nz, h);
  tm_mul(t3, t1, r, nz, h);
  tm_add(&dx[6], t2, t3, nz);
  tm_mul(t1, cphi, q, nz, h);
  tm_mul(t2, sphi, r, nz, h);
  tm_sub(&dx[7], t1, t2, nz);
  tm_inv(ic, cth, nz, h, thrown);
  tm_mul(t1, sphi, ic, nz, h);
  tm_mul(t2, t1, q, nz, h);
  tm_inv(ic, cth, nz, h, thrown);
  tm_mul(t1, cphi, ic, nz, h);
  tm_mul(t3, t1, r, nz, h);
  tm_add(&dx[8], t2, t3, nz);
  tm_mul(t1, q, r, nz, h);
  tm_smul(t1, dc((jy - jz) / jx), t1, nz);
  tm_smul(t2, dc(1.0 / jx), &u[1], nz);
  tm_add(&dx[9], t1, t2, nz);
  tm_mul(t1, p, r, nz, h);
  tm_smul(t1, dc((jz - jx) / jy), t1, nz);
  tm_smul(t2, dc(1.0 / jy), &u[2], nz);
  tm_add(&dx[10], t1, t2, nz);
  tm_mul(t1, p, q, nz, h);
  tm_smul(t1, dc((jx - jy) / jz), t1, nz);
  tm_smul(t2, dc(1.0 / jz), &u[3], nz);
  tm_add(&dx[11], t1, t2, nz);
}

// make_augmented_field(12, 4, quadrotor_ode) (fields.hpp:96-107): udot = 0
__device__ __forceinline__ void field_eval(Work& W, const TM* x, TM* dx, const double* prm, int nz, double h,
                                           bool& thrown) {
  quad_body(x, &x[12], dx, prm, W.t, nz, h, thrown);
  for (int i = 12; i < 16; ++i) tm_const(&dx[i], dc(0.0), nz);
}

__device__ __forceinline__ int ct_nz(const Work& W) {
  int z = W.p0;
  for (int q = 0; q < W.nq; ++q) z += W.wid[q];
  return z;
}

// fold_overflow's box-hull branch (flowpipe_ct.hpp:347-348) + popping the oldest block
__device__ void fold_hull(Work& W, int na, int window) {
  const int lane = threadIdx.x & 31;
  const int cap = window > 0 ? window : 1;
  while (W.nq > cap) {
    const int w = W.wid[0];
    int off_new = W.p0;
    for (int q = 0; q + 1 < W.nq; ++q) off_new += W.wid[q];
    for (int i = 0; i < na; ++i) {
      D r = dc(0.0);  // row_abs_sum of the oldest block, in column order (lane 0)
      if (lane == 0) {
        for (int j = 0; j < w; ++j) r = dadd(r, dabs(W.sM[i][W.p0 + j]));
        W.sM[i][off_new + i] = dadd(W.sM[i][off_new + i], r);
      }
    }
    __syncwarp();
    const int total = ct_nz(W);
    const int keep = total - W.p0 - w;
    for (int i = 0; i < na; ++i) {
      D tmp[MZ / 32];
#pragma unroll
      for (int k = 0; k < MZ / 32; ++k) {
        const int j = lane + 32 * k;
        if (j < keep) tmp[k] = W.sM[i][W.p0 + w + j];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < MZ / 32; ++k) {
        const int j = lane + 32 * k;
        if (j < keep) W.sM[i][W.p0 + j] = tmp[k];
      }
      __syncwarp();
    }
    if (lane == 0) {
      for (int q = 0; q + 1 < W.nq; ++q) W.wid[q] = W.wid[q + 1];
      W.nq -= 1;
    }
    __syncwarp();
  }
}

// symbolic_box (flowpipe_ct.hpp:413-424) row i: per-block row abs-sums in column order
__device__ __forceinline__ D box_radius(const Work& W, int i) {
  D r = dc(0.0);
  for (int j = 0; j < W.p0; ++j) r = dadd(r, dabs(W.sM[i][j]));
  int off = W.p0;
  for (int q = 0; q < W.nq; ++q) {
    D rq = dc(0.0);
    for (int j = 0; j < W.wid[q]; ++j) rq = dadd(rq, dabs(W.sM[i][off + j]));
    r = dadd(r, rq);
    off += W.wid[q];
  }
  return r;
}

struct FlowCfg {
  double h, eps_init, enlargement;
  int order, refine_rounds, max_enlargements, window;
};

// replay (flowpipe_ct.hpp:154-165) of p_k (W.g) with candidate remainder i0 -> i1; false = threw
__device__ bool replay(Work& W, const double* prm, int na, int nz, double h, const DI* i0, DI* i1) {
  const int lane = threadIdx.x & 31;
  // cand = p_k with remainder i0 (p_k's own remainder is zero after poly_picard)
  __syncwarp();
  if (lane == 0)
    for (int i = 0; i < na; ++i) W.g[i].rem = i0[i];
  __syncwarp();
  bool thrown = false;
  field_eval(W, W.g, W.fg, prm, nz, h, thrown);
  if (lane == 0)
    for (int i = 0; i < na; ++i) W.g[i].rem = izero();
  __syncwarp();
  if (thrown) return false;
  TM* d1 = &W.t[12];
  TM* d2 = &W.t[13];
  for (int i = 0; i < na; ++i) {
    tm_integrate(d1, &W.fg[i], nz, h);
    // seed row i: c = sc[i], az = sM[i][:], at = bz = 0, rem = 0 (rows_from_linear_tm)
    for (int j = lane; j < nz; j += 32) {
      d2->az[j] = dadd(W.sM[i][j], d1->az[j]);
      d2->bz[j] = dadd(dc(0.0), d1->bz[j]);
    }
    const Sc D1 = ld(d1);
    st(d2, Sc{dadd(W.sc[i], D1.c), dadd(dc(0.0), D1.at), iadd(izero(), D1.rem)});
    tm_sub(d2, d2, &W.g[i], nz);
    const DI r = total_range(d2, nz, h);
    __syncwarp();
    if (lane == 0) i1[i] = r;
    __syncwarp();
  }
  return true;
}

// One validated flowpipe step from the state (seed = rows of (sc, sM)); fills W.ec / W.sM (endpoint, in
// place), W.erem, W.i1 and the step box lo/hi (box_out[i] = hi - lo for the loss).  Returns the status.
__device__ int flow_step(Work& W, const double* prm, const FlowCfg& F, int na, D* width_sum, bool& box_fin) {
  const int lane = threadIdx.x & 31;
  const int nz = ct_nz(W);
  const double h = F.h;
  // poly_picard (flowpipe_ct.hpp:126-139): g = seed
  for (int i = 0; i < na; ++i) {
    for (int j = lane; j < nz; j += 32) {
      W.g[i].az[j] = W.sM[i][j];
      W.g[i].bz[j] = dc(0.0);
    }
    st(&W.g[i], Sc{W.sc[i], dc(0.0), izero()});
  }
  TM* d1 = &W.t[12];
  for (int it = 0; it < F.order; ++it) {
    bool thrown = false;
    field_eval(W, W.g, W.fg, prm, nz, h, thrown);
    if (thrown) return REACH_TUBE_TME_INV;
    for (int i = 0; i < na; ++i) {
      tm_integrate(d1, &W.fg[i], nz, h);
      for (int j = lane; j < nz; j += 32) {
        W.g[i].az[j] = dadd(W.sM[i][j], d1->az[j]);
        W.g[i].bz[j] = dadd(dc(0.0), d1->bz[j]);
      }
      const Sc D1 = ld(d1);
      st(&W.g[i], Sc{dadd(W.sc[i], D1.c), dadd(dc(0.0), D1.at), iadd(izero(), D1.rem)});
    }
  }
  for (int i = 0; i < na; ++i) {
    if (!isfinite(W.g[i].c.v)) return REACH_TUBE_PICARD_NONFINITE;
  }
  if (lane == 0)
    for (int i = 0; i < na; ++i) W.g[i].rem = izero();
  __syncwarp();
  // remainder_picard (flowpipe_ct.hpp:144-276)
  for (int i = 0; i < na; ++i) {
    W.i0[i] = DI{dc(-F.eps_init), dc(F.eps_init)};
    W.i1[i] = izero();
  }
  __syncwarp();
  bool accepted = false;
  for (int attempt = 0; attempt <= F.max_enlargements; ++attempt) {
    const bool ok = replay(W, prm, na, nz, h, W.i0, W.nx);
    if (ok && lane == 0)
      for (int i = 0; i < na; ++i) W.i1[i] = W.nx[i];
    __syncwarp();
    bool fin = true, sub = true;
    for (int i = 0; i < na; ++i) {
      fin = fin && ifin(W.i1[i]);
      sub = sub && isubset(W.i1[i], W.i0[i]);
    }
    if (ok && fin && sub) {
      accepted = true;
      break;
    }
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < na; ++i) {
        const DI induced = ok ? W.i1[i] : izero();
        const DI hull = ivalid(induced) ? ihull(W.i0[i], induced) : W.i0[i];
        const D mid = imid(hull), rad = dmul(irad(hull), dc(F.enlargement));
        W.i0[i] = DI{dsub(mid, rad), dadd(mid, rad)};
      }
    __syncwarp();
  }
  if (!accepted) return REACH_TUBE_REMAINDER;
  for (int round = 0; round < F.refine_rounds; ++round) {
    if (!replay(W, prm, na, nz, h, W.i1, W.nx)) break;
    bool fin = true, sub = true;
    for (int i = 0; i < na; ++i) {
      fin = fin && ifin(W.nx[i]);
      sub = sub && isubset(W.nx[i], W.i1[i]);
    }
    if (!(fin && sub)) break;
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < na; ++i) W.i1[i] = W.nx[i];
    __syncwarp();
  }
  // step box: tm_eval_interval(segment (p_k, rem i1), [0, h]) (taylor_model.hpp:73-97)
  {
    D wsum_all = dc(0.0);
    bool fin = true;
    for (int i = 0; i < na; ++i) {
      const Sc P = ld(&W.g[i]);
      const D lin = abs_sum(W.g[i].az, nz);
      DI acc{dsub(P.c, lin), dadd(P.c, lin)};
      acc = iadd(acc, iscale(P.at, DI{dc(0.0), dc(h)}));
      const D cross = abs_sum(W.g[i].bz, nz);
      const D tau_mag = dmax(dabs(dc(0.0)), dabs(dc(h)));
      acc = iadd(acc, DI{dneg(dmul(cross, tau_mag)), dmul(cross, tau_mag)});
      acc = iadd(acc, W.i1[i]);
      fin = fin && ifin(acc);
      wsum_all = dadd(wsum_all, dsub(acc.hi, acc.lo));  // box_volume_proxy: sum of widths in dim order
    }
    *width_sum = wsum_all;
    box_fin = fin;
  }
  // endpoint by exact integration at tau = h (flowpipe_ct.hpp:236-263), written in place over the seed
  bool exact_ok = true;
  {
    bool thrown = false;
    __syncwarp();
    if (lane == 0)
      for (int i = 0; i < na; ++i) W.g[i].rem = W.i1[i];
    __syncwarp();
    field_eval(W, W.g, W.fg, prm, nz, h, thrown);
    if (lane == 0)
      for (int i = 0; i < na; ++i) W.g[i].rem = izero();
    __syncwarp();
    if (thrown) exact_ok = false;
    if (exact_ok) {
      const D hh = dc(h);
      for (int i = 0; i < na; ++i) {
        const Sc f = ld(&W.fg[i]);
        const D ec = dadd(W.sc[i], dmul(hh, dadd(f.c, dmul(dmul(f.at, hh), dc(0.5)))));
        const DI er = iadd(imul(DI{hh, hh}, f.rem), izero());
        exact_ok = exact_ok && isfinite(ec.v) && ifin(er);
        __syncwarp();
        if (lane == 0) {
          W.ec[i] = ec;
          W.erem[i] = er;
        }
        __syncwarp();
      }
    }
  }
  if (exact_ok) {
    const D hh = dc(h);
    for (int i = 0; i < na; ++i)
      for (int j = lane; j < nz; j += 32)
        W.sM[i][j] = dadd(W.sM[i][j], dmul(hh, dadd(W.fg[i].az[j], dmul(dmul(W.fg[i].bz[j], hh), dc(0.5)))));
  } else {  // fallback: the certified segment at tau = h (:264-274)
    for (int i = 0; i < na; ++i) {
      const Sc P = ld(&W.g[i]);
      for (int j = lane; j < nz; j += 32) W.sM[i][j] = dadd(W.g[i].az[j], dmul(W.g[i].bz[j], dc(h)));
      __syncwarp();
      if (lane == 0) {
        W.ec[i] = dadd(P.c, dmul(P.at, dc(h)));
        W.erem[i] = W.i1[i];
      }
    }
  }
  __syncwarp();
  return REACH_TUBE_OK;
}

// symbolic_step (flowpipe_ct.hpp:378-409): the endpoint (already in sM) + a fresh diagonal block, fold
__device__ void symbolic_step(Work& W, int na, int window) {
  const int lane = threadIdx.x & 31;
  const int nz = ct_nz(W);
  for (int i = 0; i < na; ++i)
    for (int j = lane; j < na; j += 32) W.sM[i][nz + j] = (i == j) ? irad(W.erem[i]) : dc(0.0);
  __syncwarp();
  if (lane == 0) {
    for (int i = 0; i < na; ++i) W.sc[i] = dadd(W.ec[i], imid(W.erem[i]));
    W.wid[W.nq++] = na;
  }
  __syncwarp();
  fold_hull(W, na, window);
}

// ctl_crown (neural.hpp:398-424): the controller with y_ref folded into the first-layer bias, certified
// on the state TM x = xc + sM[0..n) z (zero remainder).  Writes u's rows into sM[n..n+l), u's centre to
// cc.uc, its remainder to cc.urem.  Returns 0, 1 (non-finite preactivation: "certification failed").
__device__ int ctl_certify(Work& W, const dual::NetView& net, int n, int l, int nz, const double* yref, int rdim) {
  const int lane = threadIdx.x & 31;
  const DevNet& N = net.N;
  const int L = N.L;
  auto& C = W.cc;
  // freeze_trailing_inputs: b0_i = b_i + sum_j W0[i][n + j] * y_j
  const int h0 = N.dims[1];
  for (int i = lane; i < h0; i += 32) {
    D b = net.b(0, i);
    for (int j = 0; j < rdim; ++j) b = dadd(b, dmul(net.w(0, i, n + j), dc(yref[j])));
    C.b0[i] = b;
  }
  // prepend layer IBP (neural.hpp:360-373): pre0_i = sum_j iv_scale(A_ij, [-1,1]) + c_i
  for (int i = lane; i < n; i += 32) {
    DI acc = izero();
    for (int j = 0; j < nz; ++j) acc = iadd(acc, iscale(W.sM[i][j], DI{dc(-1.0), dc(1.0)}));
    C.pre[0][i] = iadd(acc, ipt(C.xc[i]));
    C.hb[0][i] = C.pre[0][i];
  }
  __syncwarp();
  // IBP through the net (box_affine_image, interval.hpp:284-295); the output layer's box is unused
  int cur = 0;
  for (int l2 = 0; l2 + 1 < L; ++l2) {
    const int rows = N.dims[l2 + 1], cols = (l2 == 0) ? n : N.dims[l2];
    for (int i = lane; i < rows; i += 32) {
      DI acc = izero();
      for (int j = 0; j < cols; ++j) acc = iadd(acc, iscale(net.w(l2, i, j), C.hb[cur][j]));
      const D bi = (l2 == 0) ? C.b0[i] : net.b(l2, i);
      const DI p = iadd(acc, ipt(bi));
      C.pre[l2 + 1][i] = p;
      C.hb[cur ^ 1][i] = dual::act_d(N.acts[l2], p);
    }
    cur ^= 1;
    __syncwarp();
  }
  // CROWN backward (neural.hpp:297-327) through the wide net [prepend | net]
  const int n_o = l;
  for (int i = 0; i < n_o; ++i)
    for (int j = lane; j < n_o; j += 32) C.a[i][j] = dc(i == j ? 1.0 : 0.0);
  if (lane < n_o) {
    C.blo[lane] = dc(0.0);
    C.bup[lane] = dc(0.0);
  }
  __syncwarp();
  int acols = n_o;
  bool bad = false;
  for (int wl = L; wl >= 0; --wl) {
    const int act = (wl == 0) ? REACH_ACT_IDENTITY : N.acts[wl - 1];
    const int cols = (wl == 0) ? nz + n : ((wl == 1) ? n : N.dims[wl - 1]);
    if (act != REACH_ACT_IDENTITY) {
      bool boundary = false;
      for (int j = lane; j < acols; j += 32) {
        D s, li, ui;
        if (!dual::relax_d(act, C.pre[wl][j], s, li, ui, boundary)) bad = true;
        C.sl[j] = s;
        C.li[j] = li;
        C.ui[j] = ui;
      }
      bad = __any_sync(0xffffffffu, bad);
      if (bad) return 1;
      __syncwarp();
      if (lane < n_o) {
        const int i = lane;
        D bl = C.blo[i], bu = C.bup[i];
        for (int j = 0; j < acols; ++j) {
          const D aij = C.a[i][j];
          if (aij.v >= 0.0) {
            bl = dadd(bl, dmul(aij, C.li[j]));
            bu = dadd(bu, dmul(aij, C.ui[j]));
          } else {
            bl = dadd(bl, dmul(aij, C.ui[j]));
            bu = dadd(bu, dmul(aij, C.li[j]));
          }
          C.a[i][j] = dmul(aij, C.sl[j]);
        }
        C.blo[i] = bl;
        C.bup[i] = bu;
      }
      __syncwarp();
    }
    // shift = a . bias; b += shift
    if (lane < n_o) {
      const int i = lane;
      D acc = dc(0.0);
      for (int j = 0; j < acols; ++j) {
        const D bj = (wl == 0) ? C.xc[j] : (wl == 1 ? C.b0[j] : net.b(wl - 1, j));
        acc = dadd(acc, dmul(C.a[i][j], bj));
      }
      C.blo[i] = dadd(C.blo[i], acc);
      C.bup[i] = dadd(C.bup[i], acc);
    }
    __syncwarp();
    // a = a . W (linalg.hpp:53-63, i-k-j order: each output a sequential chain over k)
    for (int i = 0; i < n_o; ++i)
      for (int j = lane; j < cols; j += 32) {
        D acc = dc(0.0);
        for (int k = 0; k < acols; ++k) {
          D wkj;
          if (wl == 0) wkj = (j < nz) ? W.sM[k][j] : dc((j - nz) == k ? 1.0 : 0.0);
          else wkj = net.w(wl - 1, k, j);
          acc = dadd(acc, dmul(C.a[i][k], wkj));
        }
        C.an[i][j] = acc;
      }
    __syncwarp();
    for (int i = 0; i < n_o; ++i)
      for (int j = lane; j < cols; j += 32) C.a[i][j] = C.an[i][j];
    __syncwarp();
    acols = cols;
  }
  // tail (neural.hpp:383-391): c = mid(b), A = Lambda[:, :nz], rem = b - mid (zero input remainder)
  if (lane < n_o) {
    const int i = lane;
    const D mid = dmul(dadd(C.blo[i], C.bup[i]), dc(0.5));
    C.uc[i] = mid;
    C.urem[i] = DI{dsub(C.blo[i], mid), dsub(C.bup[i], mid)};
  }
  for (int i = 0; i < n_o; ++i)
    for (int j = lane; j < nz; j += 32) W.sM[n + i][j] = C.a[i][j];
  __syncwarp();
  return 0;
}

struct CtlLossArgs {
  DevNet net;              // controller (n + ref_dim -> l)
  int n, l, rdim, ctl_steps, k_atomic, intervalize, M, seeded;
  long long poff[kMaxLayers + 1];
  double prm[5];
  FlowCfg F;
  double eps, cap;
  const double* x0;        // [M][n] episode start states
  const double* yref;      // [M][ctl_steps][rdim]
  double* term_v;          // [passes][M]
  double* term_d;
  int* diverged;           // [M] (pass 0)
};

// One Dual cl_reach (closed_loop.hpp:76-182) from box_from_center(x0_e, eps) per (pass, episode).
__device__ void ctl_pass(const CtlLossArgs& A, Work& W, int pass, int ep) {
  const int lane = threadIdx.x & 31;
  const int n = A.n, l = A.l, na = n + l;
  dual::NetView net{A.net};
  if (A.seeded) dual::seed_param(net, A.poff, pass);
  // X0 = box_from_center(x0, S(eps)); x_tm = build_linear_tm(X0) (taylor_model.hpp:53-64)
  int nzx = n;
  for (int i = 0; i < n; ++i) {
    const D c = dc(A.x0[static_cast<size_t>(ep) * n + i]), r = dc(A.eps);
    const D lo = dsub(c, r), hi = dadd(c, r);
    for (int j = lane; j < n; j += 32) W.sM[i][j] = (i == j) ? dmul(dsub(hi, lo), dc(0.5)) : dc(0.0);
    if (lane == 0) W.cc.xc[i] = dmul(dadd(lo, hi), dc(0.5));
  }
  if (lane == 0) {
    W.p0 = n;
    W.nq = 0;
  }
  __syncwarp();
  int bw[16], nbw = 0;
  bool failed = false;
  D vol = dc(0.0);  // predicted_volume (training.hpp:87-93): boxes k >= 1
  for (int ci = 0; ci < A.ctl_steps && !failed; ++ci) {
    if (ci > 0) {
      if (A.intervalize) {  // x_tm = build_linear_tm(symbolic_box(aug)[0..n))
        D lo[MR], hi[MR];
        bool fin = true;
        for (int i = 0; i < n; ++i) {
          const D r = box_radius(W, i);
          lo[i] = dsub(W.sc[i], r);
          hi[i] = dadd(W.sc[i], r);
          fin = fin && isfinite(lo[i].v) && isfinite(hi[i].v);
        }
        if (!fin) {  // build_linear_tm throws std::invalid_argument: it escapes cl_reach (the loss throws)
          failed = true;
          break;
        }
        __syncwarp();
        for (int i = 0; i < n; ++i) {
          for (int j = lane; j < n; j += 32) W.sM[i][j] = (i == j) ? dmul(dsub(hi[i], lo[i]), dc(0.5)) : dc(0.0);
          if (lane == 0) W.cc.xc[i] = dmul(dadd(lo[i], hi[i]), dc(0.5));
        }
        nzx = n;
        nbw = 0;
        if (lane == 0) {
          W.p0 = n;
          W.nq = 0;
        }
        __syncwarp();
      } else {  // boundary_state_tm (closed_loop.hpp:51-69): rows 0..n of the state as they are
        nzx = ct_nz(W);
        nbw = W.nq;
        for (int q = 0; q < W.nq; ++q) bw[q] = W.wid[q];
        if (lane == 0)
          for (int i = 0; i < n; ++i) W.cc.xc[i] = W.sc[i];
        __syncwarp();
      }
    }
    const double* yr = A.yref ? A.yref + (static_cast<size_t>(ep) * A.ctl_steps + ci) * A.rdim : nullptr;
    if (ctl_certify(W, net, n, l, nzx, yr, yr ? A.rdim : 0)) {
      failed = true;
      break;
    }
    bool ufin = true;
    for (int d = 0; d < l; ++d) ufin = ufin && ifin(W.cc.urem[d]);
    if (!ufin) {
      failed = true;
      break;
    }
    // stacking (closed_loop.hpp:122-153): x rows stay, u rows written by ctl_certify, fresh block
    int p0 = nzx;
    for (int q = 0; q < nbw; ++q) p0 -= bw[q];
    for (int i = 0; i < na; ++i)
      for (int j = lane; j < na; j += 32)
        W.sM[i][nzx + j] = (i == j) ? (i < n ? dmul(dsub(dc(0.0), dc(0.0)), dc(0.5)) : irad(W.cc.urem[i - n])) : dc(0.0);
    __syncwarp();
    if (lane == 0) {
      for (int d = 0; d < n; ++d) W.sc[d] = dadd(W.cc.xc[d], dmul(dadd(dc(0.0), dc(0.0)), dc(0.5)));
      for (int d = 0; d < l; ++d) W.sc[n + d] = dadd(W.cc.uc[d], imid(W.cc.urem[d]));
      W.p0 = p0;
      W.nq = 0;
      for (int q = 0; q < nbw; ++q) W.wid[W.nq++] = bw[q];
      W.wid[W.nq++] = na;
    }
    __syncwarp();
    fold_hull(W, na, A.F.window);
    if (ci == 0) {  // tube.push(symbolic_box(aug)): a non-finite box 0 marks the tube diverged (tube.hpp:23-28)
      bool fin = true;
      for (int i = 0; i < na; ++i) {
        const D r = box_radius(W, i);
        fin = fin && isfinite(dsub(W.sc[i], r).v) && isfinite(dadd(W.sc[i], r).v);
      }
      if (!fin) {
        failed = true;
        break;
      }
    }
    for (int j = 0; j < A.k_atomic; ++j) {
      D wsum_k;
      bool box_fin = true;
      const int rc = flow_step(W, A.prm, A.F, na, &wsum_k, box_fin);
      if (rc != REACH_TUBE_OK || !box_fin) {
        failed = true;
        break;
      }
      vol = dadd(vol, wsum_k);
      symbolic_step(W, na, A.F.window);
    }
  }
  if (lane == 0) {
    D term;
    if (failed) {
      term = dc(A.cap);
    } else {
      const D a = dadd(dc(1.0), vol);
      term = D{log(a.v), __ddiv_rn(a.d, a.v)};  // reach::log (scalar.hpp:47)
    }
    const size_t o = static_cast<size_t>(pass) * A.M + ep;
    A.term_v[o] = term.v;
    A.term_d[o] = term.d;
    if (pass == 0) A.diverged[ep] = failed ? 1 : 0;
  }
  __syncwarp();
}

// Working set in shared memory: one pass per CTA (one warp per SM: the ~200 KB set fills it).
__global__ void __launch_bounds__(32, 1) ctl_reach_loss_grad_kernel(const CtlLossArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ctl_pass(A, *reinterpret_cast<Work*>(smem_raw), blockIdx.x, blockIdx.y);
}

// Working set in global memory (L1 / L2 resident), one Work slot per CTA, CTAs persistent over the
// (pass, episode) pairs: several latency-bound passes per SM instead of one.
__global__ void __launch_bounds__(32, RB_CTD_MIN_BLOCKS) ctl_reach_loss_grad_kernel_g(const CtlLossArgs A, Work* ws, long long total) {
  Work& W = ws[blockIdx.x];
  for (long long q = blockIdx.x; q < total; q += gridDim.x)
    ctl_pass(A, W, static_cast<int>(q / A.M), static_cast<int>(q % A.M));
}

}  // namespace ctd
}  // namespace rb
