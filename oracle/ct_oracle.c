/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the continuous-time closed
 * loop.  Never linked into, loaded by, or called from the product path
 * (paper_2605_25346_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs may use it.
 *
 * A plain-C restatement of cl_reach (closed_loop.hpp:76-182) with the
 * quadrotor plant: the TMExpr algebra (taylor_model.hpp:197-445), the
 * augmented analytic field (fields.hpp:96-128, systems.hpp:22-64),
 * poly_picard / remainder_picard (flowpipe_ct.hpp:126-276), the symbolic
 * state with the hull fold (flowpipe_ct.hpp:286-424), ctl_crown
 * (neural.hpp:418-424, certify_tm_input shared with reach_oracle.c), and
 * reach_with_splitting's hull (refine.hpp:121-160).  Operation for operation
 * in the reference's order with the same roundings (-ffp-contract=off) and
 * glibc's libm, so it is bit-identical to the reference compiled -O2; pinned
 * against oracle/_ref in tests/test_oracle_ct.py.
 *
 * The reference's exceptions become flags: tme_inv's domain error
 * (taylor_model.hpp:367-368) sets `thrown`; callers reproduce the reference's
 * catch sites (flowpipe_ct.hpp:186-190, 216-220, 241-263; closed_loop.hpp:160-166).
 *
 * Paths are relative to /root/reference/proj/include/reach/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_int.h"

#define CT_MAXZ 192 /* generator columns of one TM row (n + l + window * (n + l) <= 192) */
#define CT_MAXR 24  /* rows of the augmented state */

static double smin(double a, double b) { return (b < a) ? b : a; }
static double smax(double a, double b) { return (a < b) ? b : a; }

/* interval.hpp:60-94 (nearest rounding) */
static iv iv_add(iv a, iv b) { iv r = {a.lo + b.lo, a.hi + b.hi}; return r; }
static iv iv_sub(iv a, iv b) { iv r = {a.lo - b.hi, a.hi - b.lo}; return r; }
static iv iv_mul(iv a, iv b) {
  double p1 = a.lo * b.lo, p2 = a.lo * b.hi, p3 = a.hi * b.lo, p4 = a.hi * b.hi;
  iv r = {smin(smin(p1, p2), smin(p3, p4)), smax(smax(p1, p2), smax(p3, p4))};
  return r;
}
static iv iv_scale(double a, iv x) {
  iv r;
  if (a >= 0.0) { r.lo = a * x.lo; r.hi = a * x.hi; }
  else { r.lo = a * x.hi; r.hi = a * x.lo; }
  return r;
}
static iv iv_hull(iv a, iv b) { iv r = {smin(a.lo, b.lo), smax(a.hi, b.hi)}; return r; }
static iv ivp(double lo, double hi) { iv r = {lo, hi}; return r; }
static int iv_fin(iv x) { return isfinite(x.lo) && isfinite(x.hi); }
static int iv_valid(iv x) { return x.lo <= x.hi; }
static int iv_subset(iv in, iv out) { return out.lo <= in.lo && in.hi <= out.hi; }
static double iv_mid(iv x) { return (x.lo + x.hi) * 0.5; }
static double iv_rad(iv x) { return (x.hi - x.lo) * 0.5; }

/* ----------------------------------------------------------------------- */
/* TMExpr (taylor_model.hpp:197-238): one quasi-quadratic TM row.           */
typedef struct {
  double c, at;
  double az[CT_MAXZ];
  double bz[CT_MAXZ];
  iv rem;
  double h;
  int nz;
} tme;

static void tme_const(tme* r, double v, int nz, double h) {
  memset(r, 0, sizeof(*r));
  r->c = v;
  r->nz = nz;
  r->h = h;
}
static double tme_abs_z(const tme* u) { double a = 0.0; for (int j = 0; j < u->nz; ++j) a += fabs(u->az[j]); return a; }
static double tme_abs_b(const tme* u) { double a = 0.0; for (int j = 0; j < u->nz; ++j) a += fabs(u->bz[j]); return a; }
/* poly_range (taylor_model.hpp:227-235) */
static iv tme_poly_range(const tme* u) {
  double zr = tme_abs_z(u);
  iv r = {u->c - zr, u->c + zr};
  r = iv_add(r, iv_mul(ivp(0.0, u->h), ivp(u->at, u->at)));
  double br = tme_abs_b(u) * u->h;
  return iv_add(r, ivp(-br, br));
}
static iv tme_total_range(const tme* u) { return iv_add(tme_poly_range(u), u->rem); }

/* operator+ / operator- / unary - (taylor_model.hpp:245-282), elementwise in
 * the reference's operand order; r may alias a or b. */
static void tme_add(tme* r, const tme* a, const tme* b) {
  r->nz = a->nz; r->h = a->h;
  r->c = a->c + b->c;
  for (int j = 0; j < a->nz; ++j) { r->az[j] = a->az[j] + b->az[j]; r->bz[j] = a->bz[j] + b->bz[j]; }
  r->at = a->at + b->at;
  r->rem = iv_add(a->rem, b->rem);
}
static void tme_sub(tme* r, const tme* a, const tme* b) {
  r->nz = a->nz; r->h = a->h;
  r->c = a->c - b->c;
  for (int j = 0; j < a->nz; ++j) { r->az[j] = a->az[j] - b->az[j]; r->bz[j] = a->bz[j] - b->bz[j]; }
  r->at = a->at - b->at;
  r->rem = iv_sub(a->rem, b->rem);
}
/* scalar * TM (taylor_model.hpp:284-295): r.x = a.x * s; r may alias a. */
static void tme_smul(tme* r, double s, const tme* a) {
  r->nz = a->nz; r->h = a->h;
  r->rem = iv_scale(s, a->rem);
  r->c = a->c * s;
  for (int j = 0; j < a->nz; ++j) { r->az[j] = a->az[j] * s; r->bz[j] = a->bz[j] * s; }
  r->at = a->at * s;
}
/* TM + s, TM - s (taylor_model.hpp:302-317); r may alias a. */
static void tme_sadd(tme* r, const tme* a, double s) { if (r != a) *r = *a; r->c += s; }
static void tme_ssub(tme* r, const tme* a, double s) { if (r != a) *r = *a; r->c -= s; }

/* Product (taylor_model.hpp:325-360).  r must not alias u or v. */
static void tme_mul(tme* r, const tme* u, const tme* v) {
  tme_const(r, 0.0, u->nz, u->h);
  const double h = u->h;
  r->c = u->c * v->c;
  for (int j = 0; j < r->nz; ++j) {
    r->az[j] = u->c * v->az[j] + v->c * u->az[j];
    r->bz[j] = u->c * v->bz[j] + v->c * u->bz[j] + u->at * v->az[j] + v->at * u->az[j];
  }
  r->at = u->c * v->at + v->c * u->at;
  double au = tme_abs_z(u), av = tme_abs_z(v);
  double bu = tme_abs_b(u), bv = tme_abs_b(v);
  double atu = fabs(u->at), atv = fabs(v->at);
  double sym = au * av;
  sym += (au * bv + av * bu) * h;
  sym += bu * bv * h * h;
  sym += (atu * bv + atv * bu) * h * h;
  r->rem = iv_add(r->rem, ivp(-sym, sym));
  double tt = u->at * v->at;
  r->rem = iv_add(r->rem, iv_mul(ivp(0.0, h * h), ivp(tt, tt)));
  iv pu = tme_poly_range(u), pv = tme_poly_range(v);
  r->rem = iv_add(r->rem, iv_mul(pu, v->rem));
  r->rem = iv_add(r->rem, iv_mul(pv, u->rem));
  r->rem = iv_add(r->rem, iv_mul(u->rem, v->rem));
}

/* tme_inv (taylor_model.hpp:364-380); sets *thrown on a zero-containing range. */
static void tme_inv(tme* r, const tme* v, int* thrown) {
  iv range = tme_total_range(v);
  if (range.lo <= 0.0 && range.hi >= 0.0) *thrown = 1;
  double m = v->c;
  double e_lo = 1.0 / range.lo - (2.0 / m - range.lo / (m * m));
  double e_hi = 1.0 / range.hi - (2.0 / m - range.hi / (m * m));
  iv e = {smin(smin(e_lo, e_hi), 0.0), smax(smax(e_lo, e_hi), 0.0)};
  tme_smul(r, -1.0 / (m * m), v);
  tme_sadd(r, r, 2.0 / m);
  r->rem = iv_add(r->rem, e);
}

/* sin / cos (taylor_model.hpp:397-425); r must not alias u. */
static void tme_sin(tme* r, const tme* u) {
  double m = u->c;
  iv range = tme_total_range(u);
  double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
  double err = rad * rad * 0.5;
  tme_ssub(r, u, m);
  tme_smul(r, cos(m), r);
  tme_sadd(r, r, sin(m));
  r->rem = iv_add(r->rem, ivp(-err, err));
}
static void tme_cos(tme* r, const tme* u) {
  double m = u->c;
  iv range = tme_total_range(u);
  double rad = smax(fabs(range.lo - m), fabs(range.hi - m));
  double err = rad * rad * 0.5;
  tme_ssub(r, u, m);
  tme_smul(r, -sin(m), r);
  tme_sadd(r, r, cos(m));
  r->rem = iv_add(r->rem, ivp(-err, err));
}

/* tme_integrate (taylor_model.hpp:429-445); r must not alias u. */
static void tme_integrate(tme* r, const tme* u) {
  tme_const(r, 0.0, u->nz, u->h);
  const double h = u->h;
  r->at = u->c;
  for (int j = 0; j < r->nz; ++j) r->bz[j] = u->az[j];
  double half_at = u->at * 0.5;
  r->rem = iv_add(r->rem, iv_mul(ivp(0.0, h * h), ivp(half_at, half_at)));
  double bb = tme_abs_b(u) * h * h * 0.5;
  r->rem = iv_add(r->rem, ivp(-bb, bb));
  r->rem = iv_add(r->rem, iv_mul(u->rem, ivp(0.0, h)));
}

/* ----------------------------------------------------------------------- */
/* quadrotor_ode (systems.hpp:24-64) on TM rows: x 12 state rows, u 4 input  */
/* rows (the augmented (x, u) rows, fields.hpp:96-107, or held constants,    */
/* fields.hpp:20-32), dx 12 rows.  prm: mass, g, jx, jy, jz.                 */
typedef struct { tme t[12]; tme u[4]; } qscratch;

/* Field evaluations so far (work accounting for the roofline, not part of the algorithm). */
long long orc_ct_field_evals = 0;

static void quad_body(const tme* x, const tme* u, tme* dx, const double* prm, qscratch* s, int* thrown) {
  ++orc_ct_field_evals;
  const double mass = prm[0], grav = prm[1], jx = prm[2], jy = prm[3], jz = prm[4];
  const int nz = x[0].nz;
  const double h = x[0].h;
  tme *sphi = &s->t[0], *cphi = &s->t[1], *sth = &s->t[2], *cth = &s->t[3], *spsi = &s->t[4], *cpsi = &s->t[5];
  tme *a = &s->t[6], *t1 = &s->t[7], *t2 = &s->t[8], *t3 = &s->t[9], *ic = &s->t[10], *tth = &s->t[11];
  const tme *phi = &x[6], *theta = &x[7], *psi = &x[8], *p = &x[9], *q = &x[10], *r = &x[11];
  tme_sin(sphi, phi); tme_cos(cphi, phi);
  tme_sin(sth, theta); tme_cos(cth, theta);
  tme_sin(spsi, psi); tme_cos(cpsi, psi);
  /* b3x = cphi*sth*cpsi + sphi*spsi ; dx3 = a * b3x */
  tme_smul(a, 1.0 / mass, &u[0]);
  dx[0] = x[3]; dx[1] = x[4]; dx[2] = x[5];
  tme_mul(t1, cphi, sth); tme_mul(t2, t1, cpsi); tme_mul(t3, sphi, spsi); tme_add(t2, t2, t3);
  tme_mul(&dx[3], a, t2);
  tme_mul(t2, t1, spsi); tme_mul(t3, sphi, cpsi); tme_sub(t2, t2, t3);
  tme_mul(&dx[4], a, t2);
  tme_mul(t2, cphi, cth); tme_mul(t3, a, t2); tme_ssub(&dx[5], t3, grav);
  /* tth = sth / cth */
  tme_inv(ic, cth, thrown);
  tme_mul(tth, sth, ic);
  /* dx6 = p + sphi*tth*q + cphi*tth*r */
  tme_mul(t1, sphi, tth); tme_mul(t2, t1, q); tme_add(t2, p, t2);
  tme_mul(t1, cphi, tth); tme_mul(t3, t1, r); tme_add(&dx[6], t2, t3);
  /* dx7 = cphi*q - sphi*r */
  tme_mul(t1, cphi, q); tme_mul(t2, sphi, r); tme_sub(&dx[7], t1, t2);
  /* dx8 = (sphi/cth)*q + (cphi/cth)*r ; each / re-evaluates tme_inv(cth) */
  tme_inv(ic, cth, thrown);
  tme_mul(t1, sphi, ic); tme_mul(t2, t1, q);
  tme_inv(ic, cth, thrown);
  tme_mul(t1, cphi, ic); tme_mul(t3, t1, r); tme_add(&dx[8], t2, t3);
  /* dx9..11 */
  tme_mul(t1, q, r); tme_smul(t1, (jy - jz) / jx, t1); tme_smul(t2, 1.0 / jx, &u[1]); tme_add(&dx[9], t1, t2);
  tme_mul(t1, p, r); tme_smul(t1, (jz - jx) / jy, t1); tme_smul(t2, 1.0 / jy, &u[2]); tme_add(&dx[10], t1, t2);
  tme_mul(t1, p, q); tme_smul(t1, (jx - jy) / jz, t1); tme_smul(t2, 1.0 / jz, &u[3]); tme_add(&dx[11], t1, t2);
  (void)nz; (void)h;
}

/* The fields of fields.hpp that run on the device. */
#define CTF_QUAD_AUG 100 /* make_augmented_field(12, 4, quadrotor_ode): 16 rows */
typedef struct { int kind; int n; const double* params; } ctfield;

static void field_eval(const ctfield* F, const tme* x, tme* dx, qscratch* s, int* thrown) {
  const int nz = x[0].nz;
  const double h = x[0].h;
  switch (F->kind) {
    case CTF_QUAD_AUG: /* fields.hpp:96-107: (x, u) rows, udot = 0 */
      quad_body(x, &x[12], dx, F->params, s, thrown);
      for (int i = 12; i < 16; ++i) tme_const(&dx[i], 0.0, nz, h);
      break;
    case REACH_FIELD_QUADROTOR: /* quadrotor_field (fields.hpp:51-56): held input rows tme_const(u) */
      for (int k = 0; k < 4; ++k) tme_const(&s->u[k], F->params[5 + k], nz, h);
      quad_body(x, s->u, dx, F->params, s, thrown);
      break;
    case REACH_FIELD_ZERO: /* dx.assign(n, x[0] * 0.0) (fields.hpp:90) */
      ++orc_ct_field_evals;
      for (int i = 0; i < F->n; ++i) tme_smul(&dx[i], 0.0, &x[0]);
      break;
    case REACH_FIELD_DIAG_LINEAR: /* diag_linear_ode (systems.hpp:154-159) */
      ++orc_ct_field_evals;
      for (int i = 0; i < F->n; ++i) tme_smul(&dx[i], F->params[i], &x[i]);
      break;
    case REACH_FIELD_ROTATION: /* rotation_ode (systems.hpp:162-167) */
      ++orc_ct_field_evals;
      tme_smul(&dx[0], -F->params[0], &x[1]);
      tme_smul(&dx[1], F->params[0], &x[0]);
      break;
  }
}


/* ----------------------------------------------------------------------- */
/* Symbolic state (flowpipe_ct.hpp:286-300): x = c + [G0 | Q1 .. Qnq] y.    */
typedef struct {
  int na, p0, nq, window;
  double c[CT_MAXR];
  double M[CT_MAXR][CT_MAXZ];
  int wid[16];
} ctsym;

static int ct_nz(const ctsym* s) { int z = s->p0; for (int q = 0; q < s->nq; ++q) z += s->wid[q]; return z; }

/* fold_overflow (flowpipe_ct.hpp:317-350).  Square G0 (ct_reach): absorb the
 * oldest block into G0's frame when G0^-1 Q is bounded (:326-346); else (and
 * always in cl_reach, where G0 is (n+l) x n) the box-hull fallback (:347-348). */
static void ct_fold(ctsym* s) {
  const int cap = s->window > 0 ? s->window : 1;
  const int n = s->na;
  while (s->nq > cap) {
    const int w = s->wid[0];
    int off_new = s->p0;
    for (int q = 0; q + 1 < s->nq; ++q) off_new += s->wid[q];
    int folded = 0;
    if (s->p0 == n) {
      double g0[CT_MAXR * CT_MAXR], a[CT_MAXR * CT_MAXR], x[CT_MAXR * CT_MAXR], e[CT_MAXR * CT_MAXR], r[CT_MAXR];
      for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) g0[i * n + j] = s->M[i][j];
        for (int j = 0; j < w; ++j) a[i * w + j] = s->M[i][n + j];
      }
      if (orc_i_mat_solve(n, w, g0, a, x)) {
        double worst = 0.0;
        for (int j = 0; j < n; ++j) {
          double rs = 0.0;
          for (int k = 0; k < w; ++k) rs += fabs(x[j * w + k]);
          r[j] = rs * (1.0 + 1e-12);
          worst = smax(worst, r[j]);
        }
        if (worst <= 1.0) {
          for (int i = 0; i < n; ++i) {
            for (int j = 0; j < w; ++j) e[i * w + j] = 0.0;
            for (int k = 0; k < n; ++k)
              for (int j = 0; j < w; ++j) e[i * w + j] += g0[i * n + k] * x[k * w + j];
          }
          for (int i = 0; i < n; ++i)
            for (int j = 0; j < w; ++j) e[i * w + j] -= a[i * w + j];
          for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) s->M[i][j] *= 1.0 + r[j];
          for (int i = 0; i < n; ++i) {
            double rs = 0.0;
            for (int j = 0; j < w; ++j) rs += fabs(e[i * w + j]);
            s->M[i][off_new + i] += rs * (1.0 + 1e-12);
          }
          folded = 1;
        }
      }
    }
    for (int i = 0; !folded && i < s->na; ++i) {
      double r = 0.0;
      for (int j = 0; j < w; ++j) r += fabs(s->M[i][s->p0 + j]);
      s->M[i][off_new + i] += r;
    }
    const int total = ct_nz(s);
    const int keep = total - s->p0 - w;
    for (int i = 0; keep > 0 && i < s->na; ++i)
      memmove(&s->M[i][s->p0], &s->M[i][s->p0 + w], sizeof(double) * (size_t)keep);
    memmove(s->wid, s->wid + 1, sizeof(int) * (size_t)(s->nq - 1));
    s->nq -= 1;
  }
}

/* symbolic_box (flowpipe_ct.hpp:413-424); returns 1 if finite. */
static int ct_box(const ctsym* s, double* lo, double* hi) {
  int fin = 1;
  for (int i = 0; i < s->na; ++i) {
    double r = 0.0;
    for (int j = 0; j < s->p0; ++j) r += fabs(s->M[i][j]);
    int off = s->p0;
    for (int q = 0; q < s->nq; ++q) {
      double rq = 0.0;
      for (int j = 0; j < s->wid[q]; ++j) rq += fabs(s->M[i][off + j]);
      r += rq;
      off += s->wid[q];
    }
    lo[i] = s->c[i] - r;
    hi[i] = s->c[i] + r;
    if (!isfinite(lo[i]) || !isfinite(hi[i])) fin = 0;
  }
  return fin;
}

/* ----------------------------------------------------------------------- */
/* One validated flowpipe step (poly_picard + remainder_picard,             */
/* flowpipe_ct.hpp:126-276) from the symbolic seed of `s` (:353-370).       */
typedef struct {
  tme seed[CT_MAXR], pk[CT_MAXR], g[CT_MAXR], fg[CT_MAXR], cand[CT_MAXR];
  tme d1, d2;
  qscratch q;
} ctwork;

typedef struct {
  iv i1[CT_MAXR];
  double ec[CT_MAXR];
  double eA[CT_MAXR][CT_MAXZ];
  iv erem[CT_MAXR];
} ctstep;

/* replay (flowpipe_ct.hpp:154-165): I1 induced by candidate remainder i0. */
static int ct_replay(ctwork* w, const ctfield* F, int na, const iv* i0, iv* i1) {
  int thrown = 0;
  for (int i = 0; i < na; ++i) { w->cand[i] = w->pk[i]; w->cand[i].rem = i0[i]; }
  field_eval(F, w->cand, w->fg, &w->q, &thrown);
  if (thrown) return 1;
  for (int i = 0; i < na; ++i) {
    tme_integrate(&w->d1, &w->fg[i]);
    tme_add(&w->d2, &w->seed[i], &w->d1);
    tme_sub(&w->d2, &w->d2, &w->pk[i]);
    i1[i] = tme_total_range(&w->d2);
  }
  return 0;
}

static int box_finite(const iv* b, int n) { for (int i = 0; i < n; ++i) if (!iv_fin(b[i])) return 0; return 1; }
static int box_subset(const iv* in, const iv* out, int n) {
  for (int i = 0; i < n; ++i) if (!iv_subset(in[i], out[i])) return 0;
  return 1;
}

/* Returns REACH_TUBE_OK, or the failure status.  Fills st (segment remainder
 * i1, endpoint) and the step box lo/hi (tm_eval_interval, taylor_model.hpp:73-97). */
static int ct_flow_step(const ctsym* s, const reach_flowpipe_params* fp, const ctfield* F, ctwork* w, ctstep* st,
                        double* blo, double* bhi, int* box_fin) {
  const int na = s->na, nz = ct_nz(s);
  const double h = fp->h;
  /* seed rows (rows_from_linear_tm, flowpipe_ct.hpp:89-100) */
  for (int i = 0; i < na; ++i) {
    tme_const(&w->seed[i], s->c[i], nz, h);
    for (int j = 0; j < nz; ++j) w->seed[i].az[j] = s->M[i][j];
  }
  /* poly_picard (flowpipe_ct.hpp:126-139) */
  for (int i = 0; i < na; ++i) w->g[i] = w->seed[i];
  for (int it = 0; it < fp->order; ++it) {
    int thrown = 0;
    field_eval(F, w->g, w->fg, &w->q, &thrown);
    if (thrown) return REACH_TUBE_TME_INV;
    for (int i = 0; i < na; ++i) {
      tme_integrate(&w->d1, &w->fg[i]);
      tme_add(&w->g[i], &w->seed[i], &w->d1);
    }
  }
  for (int i = 0; i < na; ++i) {
    if (!isfinite(w->g[i].c)) return REACH_TUBE_PICARD_NONFINITE;
    w->g[i].rem = ivp(0.0, 0.0);
  }
  for (int i = 0; i < na; ++i) w->pk[i] = w->g[i];
  /* remainder_picard (flowpipe_ct.hpp:144-276) */
  iv i0[CT_MAXR], i1[CT_MAXR], nx[CT_MAXR];
  for (int i = 0; i < na; ++i) { i0[i] = ivp(-fp->eps_init, fp->eps_init); i1[i] = ivp(0.0, 0.0); }
  int accepted = 0;
  for (int attempt = 0; attempt <= fp->max_enlargements; ++attempt) {
    int threw = ct_replay(w, F, na, i0, nx);
    if (!threw) memcpy(i1, nx, sizeof(iv) * (size_t)na);
    if (!threw && box_finite(i1, na) && box_subset(i1, i0, na)) { accepted = 1; break; }
    for (int i = 0; i < na; ++i) {
      iv induced = threw ? ivp(0.0, 0.0) : i1[i];
      iv hull = iv_valid(induced) ? iv_hull(i0[i], induced) : i0[i];
      double mid = iv_mid(hull), rad = iv_rad(hull) * fp->enlargement;
      i0[i] = ivp(mid - rad, mid + rad);
    }
  }
  if (!accepted) return REACH_TUBE_REMAINDER;
  for (int round = 0; round < fp->refine_rounds; ++round) {
    if (ct_replay(w, F, na, i1, nx)) break;
    if (!(box_finite(nx, na) && box_subset(nx, i1, na))) break;
    memcpy(i1, nx, sizeof(iv) * (size_t)na);
  }
  memcpy(st->i1, i1, sizeof(iv) * (size_t)na);
  /* endpoint by exact integration at tau = h (flowpipe_ct.hpp:236-263) */
  int exact_ok = 1;
  {
    int thrown = 0;
    for (int i = 0; i < na; ++i) { w->cand[i] = w->pk[i]; w->cand[i].rem = i1[i]; }
    field_eval(F, w->cand, w->fg, &w->q, &thrown);
    if (thrown) exact_ok = 0;
    const double hh = h;
    for (int i = 0; exact_ok && i < na; ++i) {
      const tme* f = &w->fg[i];
      const tme* s0 = &w->seed[i];
      st->ec[i] = s0->c + hh * (f->c + f->at * hh * 0.5);
      for (int j = 0; j < nz; ++j) st->eA[i][j] = s0->az[j] + hh * (f->az[j] + f->bz[j] * hh * 0.5);
      st->erem[i] = iv_add(iv_mul(ivp(hh, hh), f->rem), s0->rem);
    }
    if (exact_ok) {
      exact_ok = box_finite(st->erem, na);
      for (int i = 0; exact_ok && i < na; ++i) if (!isfinite(st->ec[i])) exact_ok = 0;
    }
  }
  if (!exact_ok) { /* fallback: the certified segment at tau = h (:264-274) */
    for (int i = 0; i < na; ++i) {
      st->ec[i] = w->pk[i].c + w->pk[i].at * h;
      for (int j = 0; j < nz; ++j) st->eA[i][j] = w->pk[i].az[j] + w->pk[i].bz[j] * h;
      st->erem[i] = i1[i];
    }
  }
  /* tm_eval_interval(segment, [0, h]) */
  int fin = 1;
  for (int i = 0; i < na; ++i) {
    const tme* p = &w->pk[i];
    double lin = 0.0;
    for (int j = 0; j < nz; ++j) lin += fabs(p->az[j]);
    iv acc = {p->c - lin, p->c + lin};
    acc = iv_add(acc, iv_scale(p->at, ivp(0.0, h)));
    double cross = 0.0;
    for (int j = 0; j < nz; ++j) cross += fabs(p->bz[j]);
    double tau_mag = smax(fabs(0.0), fabs(h));
    acc = iv_add(acc, ivp(-cross * tau_mag, cross * tau_mag));
    acc = iv_add(acc, i1[i]);
    blo[i] = acc.lo;
    bhi[i] = acc.hi;
    if (!iv_fin(acc)) fin = 0;
  }
  *box_fin = fin;
  return REACH_TUBE_OK;
}

/* symbolic_step (flowpipe_ct.hpp:378-409) */
static void ct_symbolic_step(ctsym* s, const ctstep* st) {
  const int na = s->na, nz = ct_nz(s);
  for (int i = 0; i < na; ++i) {
    s->c[i] = st->ec[i] + iv_mid(st->erem[i]);
    for (int j = 0; j < nz; ++j) s->M[i][j] = st->eA[i][j];
    for (int j = 0; j < na; ++j) s->M[i][nz + j] = (i == j) ? iv_rad(st->erem[i]) : 0.0;
  }
  s->wid[s->nq++] = na;
  ct_fold(s);
}

/* ----------------------------------------------------------------------- */
/* cl_reach (closed_loop.hpp:76-182) for one initial box.  lo/hi receive up
 * to 1 + ctl_steps * k_atomic boxes of n + l dims; returns the box count. */
static int cl_one(const net_t* ctl, const reach_cl_spec* sp, const double* x0lo, const double* x0hi, double* lo,
                  double* hi, int* failed_step, int* status) {
  const int n = sp->n, l = sp->l, na = n + l, K = sp->k_atomic;
  ctsym* s = (ctsym*)calloc(1, sizeof(ctsym));
  ctwork* w = (ctwork*)malloc(sizeof(ctwork));
  ctstep* st = (ctstep*)malloc(sizeof(ctstep));
  double* xA = (double*)malloc(sizeof(double) * (size_t)n * CT_MAXZ);
  double* uA = (double*)malloc(sizeof(double) * (size_t)l * CT_MAXZ);
  double xc[CT_MAXR], uc[CT_MAXR];
  iv urem[CT_MAXR], ig[CT_MAXR];
  memset(ig, 0, sizeof(ig));
  /* frozen controller (freeze_trailing_inputs, neural.hpp:398-413) per control step */
  const layer_t* l0 = &ctl->layers[0];
  double* w0 = (double*)malloc(sizeof(double) * (size_t)l0->rows * n);
  double* b0 = (double*)malloc(sizeof(double) * (size_t)l0->rows);
  layer_t* fl = (layer_t*)malloc(sizeof(layer_t) * (size_t)ctl->n_layers);
  memcpy(fl, ctl->layers, sizeof(layer_t) * (size_t)ctl->n_layers);
  net_t fz = {ctl->n_layers, fl};
  for (int i = 0; i < l0->rows; ++i)
    for (int j = 0; j < n; ++j) w0[(size_t)i * n + j] = l0->w[(size_t)i * l0->cols + j];
  fl[0].cols = n;
  fl[0].w = w0;
  fl[0].b = b0;

  *failed_step = -1;
  *status = REACH_TUBE_OK;
  int nb = 0, gstep = 0;
  s->window = sp->fp.window;
  s->na = na;
  /* x_tm = build_linear_tm(x0) (taylor_model.hpp:53-64) */
  int nzx = n, nbw = 0;
  int bw[16];
  for (int i = 0; i < n; ++i) {
    xc[i] = (x0lo[i] + x0hi[i]) * 0.5;
    for (int j = 0; j < n; ++j) xA[(size_t)i * nzx + j] = (i == j) ? (x0hi[i] - x0lo[i]) * 0.5 : 0.0;
  }
  for (int ci = 0; ci < sp->ctl_steps; ++ci) {
    if (ci > 0) {
      if (sp->intervalize_boundary) {
        double blo[CT_MAXR], bhi[CT_MAXR];
        ct_box(s, blo, bhi);
        int xfin = 1;
        for (int i = 0; i < n; ++i) if (!isfinite(blo[i]) || !isfinite(bhi[i])) xfin = 0;
        if (!xfin) { /* build_linear_tm throws std::invalid_argument: it escapes cl_reach */
          *failed_step = 0; *status = REACH_TUBE_OTHER; nb = 0; goto done;
        }
        nzx = n; nbw = 0;
        for (int i = 0; i < n; ++i) {
          xc[i] = (blo[i] + bhi[i]) * 0.5;
          for (int j = 0; j < n; ++j) xA[(size_t)i * nzx + j] = (i == j) ? (bhi[i] - blo[i]) * 0.5 : 0.0;
        }
      } else { /* boundary_state_tm (closed_loop.hpp:51-69) */
        nzx = ct_nz(s);
        for (int i = 0; i < n; ++i) {
          xc[i] = s->c[i];
          for (int j = 0; j < nzx; ++j) xA[(size_t)i * nzx + j] = s->M[i][j];
        }
        nbw = s->nq;
        for (int q = 0; q < s->nq; ++q) bw[q] = s->wid[q];
      }
    }
    /* ctl_crown (neural.hpp:418-424) */
    for (int i = 0; i < l0->rows; ++i) {
      double b = l0->b[i];
      for (int j = 0; j < sp->ref_dim; ++j) b += l0->w[(size_t)i * l0->cols + n + j] * sp->y_ref[(size_t)ci * sp->ref_dim + j];
      b0[i] = b;
    }
    if (orc_i_certify_tm_input(&fz, n, nzx, xc, xA, ig, uc, uA, urem)) {
      *failed_step = gstep; *status = REACH_TUBE_CTL_FAILED; goto done;
    }
    if (!box_finite(urem, l)) { *failed_step = gstep; *status = REACH_TUBE_CTL_DIVERGED; goto done; }
    /* stacking (closed_loop.hpp:122-153) */
    {
      int p0 = nzx;
      for (int q = 0; q < nbw; ++q) p0 -= bw[q];
      memset(s->M, 0, sizeof(s->M));
      for (int d = 0; d < n; ++d) {
        s->c[d] = xc[d] + (0.0 + 0.0) * 0.5;
        for (int j = 0; j < nzx; ++j) s->M[d][j] = xA[(size_t)d * nzx + j];
      }
      for (int d = 0; d < l; ++d) {
        s->c[n + d] = uc[d] + iv_mid(urem[d]);
        for (int j = 0; j < nzx; ++j) s->M[n + d][j] = uA[(size_t)d * nzx + j];
      }
      for (int d = 0; d < na; ++d) s->M[d][nzx + d] = (d < n) ? (0.0 - 0.0) * 0.5 : iv_rad(urem[d - n]);
      s->p0 = p0;
      s->nq = 0;
      for (int q = 0; q < nbw; ++q) s->wid[s->nq++] = bw[q];
      s->wid[s->nq++] = na;
      ct_fold(s);
    }
    if (ci == 0) {
      ct_box(s, lo, hi);
      nb = 1;
    }
    const ctfield F = {CTF_QUAD_AUG, na, sp->plant_params};
    for (int j = 0; j < K; ++j) {
      int fin;
      int rc = ct_flow_step(s, &sp->fp, &F, w, st, lo + (size_t)nb * na, hi + (size_t)nb * na, &fin);
      if (rc != REACH_TUBE_OK) { *failed_step = gstep; *status = rc; goto done; }
      nb += 1;
      gstep += 1;
      if (!fin) { *failed_step = gstep - 1; *status = REACH_TUBE_DIVERGED_BOX; goto done; }
      ct_symbolic_step(s, st);
    }
  }
done:
  free(s); free(w); free(st); free(xA); free(uA); free(w0); free(b0); free(fl);
  return nb;
}

int orc_cl_batch(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, int32_t batch, const double* x0_lo,
                 const double* x0_hi, const reach_tube_out* out) {
  if (sp->plant != REACH_PLANT_QUADROTOR || sp->n != 12 || sp->l != 4) return REACH_E_UNSUPPORTED;
  net_t ctl = orc_i_net_from_desc(ctl_desc);
  const int n = sp->n, na = sp->n + sp->l, T = 1 + sp->ctl_steps * sp->k_atomic;
  for (int b = 0; b < batch; ++b) {
    int fs, st;
    out->n_boxes[b] = cl_one(&ctl, sp, x0_lo + (size_t)b * n, x0_hi + (size_t)b * n, out->lo + (size_t)b * T * na,
                             out->hi + (size_t)b * T * na, &fs, &st);
    out->failed_step[b] = fs;
    out->status[b] = st;
  }
  free(ctl.layers);
  return REACH_OK;
}

/* split_box part p (refine.hpp:83-115), last dimension fastest. */
static void ct_split_part(int n, const double* xlo, const double* xhi, const int32_t* counts, int64_t p, double* lo,
                          double* hi) {
  for (int d = n - 1; d >= 0; --d) {
    int k = counts[d];
    int i = (int)(p % k);
    p /= k;
    lo[d] = (i == 0) ? xlo[d] : xlo[d] + (xhi[d] - xlo[d]) * ((double)i / k);
    hi[d] = (i + 1 == k) ? xhi[d] : xlo[d] + (xhi[d] - xlo[d]) * ((double)(i + 1) / k);
  }
}

/* reach_with_splitting(cl_reach) hull (refine.hpp:121-160) over parts [begin, end). */
int orc_cl_split_hull(const reach_net_desc* ctl_desc, const reach_cl_spec* sp, const reach_cl_split_args* a,
                      const reach_hull_out* out) {
  if (sp->plant != REACH_PLANT_QUADROTOR || sp->n != 12 || sp->l != 4) return REACH_E_UNSUPPORTED;
  const int n = sp->n, na = sp->n + sp->l, T = 1 + sp->ctl_steps * sp->k_atomic;
  int64_t total = 1;
  for (int d = 0; d < n; ++d) { if (a->counts[d] < 1) return REACH_E_INVALID_ARGUMENT; total *= a->counts[d]; }
  int64_t begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
  if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;
  net_t ctl = orc_i_net_from_desc(ctl_desc);
  double* lo = (double*)malloc(sizeof(double) * (size_t)T * na);
  double* hi = (double*)malloc(sizeof(double) * (size_t)T * na);
  double plo[CT_MAXR], phi[CT_MAXR];
  int steps = 0;
  int64_t key = INT64_MAX;
  for (int k = 0; k < T; ++k) out->box_diverged[k] = 0;
  for (int64_t p = begin; p < end; ++p) {
    ct_split_part(n, a->x0_lo, a->x0_hi, a->counts, p, plo, phi);
    int fs, st;
    int nb = cl_one(&ctl, sp, plo, phi, lo, hi, &fs, &st);
    if (p == begin) {
      steps = nb;
      for (int k = 0; k < nb * na; ++k) { out->lo[k] = lo[k]; out->hi[k] = hi[k]; }
    } else {
      int upto = nb < steps ? nb : steps;
      for (int k = 0; k < upto * na; ++k) {
        out->lo[k] = smin(out->lo[k], lo[k]);
        out->hi[k] = smax(out->hi[k], hi[k]);
      }
      if (nb < steps) steps = nb;
    }
    for (int k = 0; k < nb; ++k) {
      int fin = 1;
      for (int d = 0; d < na; ++d) if (!isfinite(lo[k * na + d]) || !isfinite(hi[k * na + d])) fin = 0;
      if (!fin) out->box_diverged[k] = 1;
    }
    if (st != REACH_TUBE_OK) {
      int64_t kk = ((int64_t)(fs >= 0 ? fs : nb) << 40) | ((int64_t)p << 8) | (int64_t)(st & 0xff);
      if (kk < key) key = kk;
    }
  }
  out->n_boxes[0] = steps;
  out->fail_key[0] = key;
  free(lo); free(hi); free(ctl.layers);
  return REACH_OK;
}

/* ----------------------------------------------------------------------- */
/* ct_reach (flowpipe_ct.hpp:428-458) of an analytic field: box 0 is X0.    */
static int ct_reach_one(const ctfield* F, const reach_flowpipe_params* fp, const double* x0lo, const double* x0hi,
                        double* lo, double* hi, int* failed_step, int* status) {
  const int n = F->n;
  ctsym* s = (ctsym*)calloc(1, sizeof(ctsym));
  ctwork* w = (ctwork*)malloc(sizeof(ctwork));
  ctstep* st = (ctstep*)malloc(sizeof(ctstep));
  *failed_step = -1;
  *status = REACH_TUBE_OK;
  for (int d = 0; d < n; ++d) { lo[d] = x0lo[d]; hi[d] = x0hi[d]; }
  int nb = 1;
  /* init_symbolic_state (flowpipe_ct.hpp:302-309) */
  s->na = n; s->p0 = n; s->nq = 0; s->window = fp->window;
  for (int i = 0; i < n; ++i) {
    s->c[i] = (x0lo[i] + x0hi[i]) * 0.5;
    s->M[i][i] = (x0hi[i] - x0lo[i]) * 0.5;
  }
  for (int step = 0; step < fp->steps; ++step) {
    int fin;
    int rc = ct_flow_step(s, fp, F, w, st, lo + (size_t)nb * n, hi + (size_t)nb * n, &fin);
    if (rc != REACH_TUBE_OK) { *failed_step = step; *status = rc; break; }
    nb += 1;
    if (!fin) { *failed_step = step; *status = REACH_TUBE_DIVERGED_BOX; break; }
    ct_symbolic_step(s, st);
  }
  free(s); free(w); free(st);
  return nb;
}

int orc_ct_batch(const reach_field_desc* fd, const reach_flowpipe_params* fp, int32_t batch, const double* x0_lo,
                 const double* x0_hi, const reach_tube_out* out) {
  const int n = fd->n, T = 1 + fp->steps;
  if (n < 1 || n > 16) return REACH_E_UNSUPPORTED;
  const ctfield F = {fd->kind, n, fd->params};
  for (int b = 0; b < batch; ++b) {
    int fs, st;
    out->n_boxes[b] = ct_reach_one(&F, fp, x0_lo + (size_t)b * n, x0_hi + (size_t)b * n, out->lo + (size_t)b * T * n,
                                   out->hi + (size_t)b * T * n, &fs, &st);
    out->failed_step[b] = fs;
    out->status[b] = st;
  }
  return REACH_OK;
}

/* reach_with_splitting(ct_reach) hull (refine.hpp:121-160) over parts [begin, end). */
int orc_ct_split_hull(const reach_field_desc* fd, const reach_flowpipe_params* fp, const reach_cl_split_args* a,
                      const reach_hull_out* out) {
  const int n = fd->n, T = 1 + fp->steps;
  if (n < 1 || n > 16) return REACH_E_UNSUPPORTED;
  int64_t total = 1;
  for (int d = 0; d < n; ++d) { if (a->counts[d] < 1) return REACH_E_INVALID_ARGUMENT; total *= a->counts[d]; }
  int64_t begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
  if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;
  const ctfield F = {fd->kind, n, fd->params};
  double* lo = (double*)malloc(sizeof(double) * (size_t)T * n);
  double* hi = (double*)malloc(sizeof(double) * (size_t)T * n);
  double plo[CT_MAXR], phi[CT_MAXR];
  int steps = 0;
  int64_t key = INT64_MAX;
  for (int k = 0; k < T; ++k) out->box_diverged[k] = 0;
  for (int64_t p = begin; p < end; ++p) {
    ct_split_part(n, a->x0_lo, a->x0_hi, a->counts, p, plo, phi);
    int fs, st;
    int nb = ct_reach_one(&F, fp, plo, phi, lo, hi, &fs, &st);
    if (p == begin) {
      steps = nb;
      for (int k = 0; k < nb * n; ++k) { out->lo[k] = lo[k]; out->hi[k] = hi[k]; }
    } else {
      int upto = nb < steps ? nb : steps;
      for (int k = 0; k < upto * n; ++k) {
        out->lo[k] = smin(out->lo[k], lo[k]);
        out->hi[k] = smax(out->hi[k], hi[k]);
      }
      if (nb < steps) steps = nb;
    }
    for (int k = 0; k < nb; ++k) {
      int fin = 1;
      for (int d = 0; d < n; ++d) if (!isfinite(lo[k * n + d]) || !isfinite(hi[k * n + d])) fin = 0;
      if (!fin) out->box_diverged[k] = 1;
    }
    if (st != REACH_TUBE_OK) {
      int64_t kk = ((int64_t)(fs >= 0 ? fs : nb) << 40) | ((int64_t)p << 8) | (int64_t)(st & 0xff);
      if (kk < key) key = kk;
    }
  }
  out->n_boxes[0] = steps;
  out->fail_key[0] = key;
  free(lo); free(hi);
  return REACH_OK;
}
