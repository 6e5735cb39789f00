/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle.  Never linked into, loaded by,
 * or called from the product path (paper_2605_25346_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
 *
 * A plain-C restatement of the reference's discrete-time reachability path,
 * operation for operation in the same order and rounding (no FMA contraction:
 * built with -ffp-contract=off), so it is bit-identical to the reference
 * compiled at -O2 on x86-64.  Pinned against oracle/_ref (the reference
 * itself) and the reference's golden vectors in tests/test_oracle.py.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/reach/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_int.h"

/* std::min / std::max semantics (first argument wins ties, NaN-asymmetric). */
static double smin(double a, double b) { return (b < a) ? b : a; }
static double smax(double a, double b) { return (a < b) ? b : a; }

/* iv_add (interval.hpp:60) in nearest rounding. */
static iv iv_add(iv a, iv b) { iv r = {a.lo + b.lo, a.hi + b.hi}; return r; }
/* iv_scale (interval.hpp:83). */
static iv iv_scale(double a, iv x) {
  iv r;
  if (a >= 0.0) { r.lo = a * x.lo; r.hi = a * x.hi; }
  else { r.lo = a * x.hi; r.hi = a * x.lo; }
  return r;
}
static int iv_finite(iv x) { return isfinite(x.lo) && isfinite(x.hi); }

static net_t net_from_desc(const reach_net_desc* d) {
  net_t net;
  net.n_layers = d->n_layers;
  net.layers = (layer_t*)malloc(sizeof(layer_t) * (size_t)d->n_layers);
  size_t k = 0;
  for (int l = 0; l < d->n_layers; ++l) {
    layer_t* L = &net.layers[l];
    L->rows = d->dims[l + 1];
    L->cols = d->dims[l];
    L->act = d->acts[l];
    L->w = d->params + k;
    k += (size_t)L->rows * L->cols;
    L->b = d->params + k;
    k += (size_t)L->rows;
  }
  return net;
}

/* relax_activation (neural.hpp:166-227).  Returns 0, or 1 on a non-finite
 * preactivation (the reference throws std::invalid_argument). */
static int relax_activation(int act, iv pre, double* slope, double* li, double* ui) {
  if (!iv_finite(pre)) return 1;
  const double l = pre.lo, u = pre.hi;
  *slope = 0.0; *li = 0.0; *ui = 0.0;
  if (act == REACH_ACT_IDENTITY) {
    *slope = 1.0;
  } else if (act == REACH_ACT_RELU) {
    if (l >= 0.0) {
      *slope = 1.0;
    } else if (u <= 0.0) {
      *slope = 0.0;
    } else {
      double s = u / (u - l);
      *slope = s;
      *ui = -s * l;
      *li = smin(0.0, smin(-s * l, u - s * u));
    }
  } else { /* tanh */
    double tl = tanh(l), tu = tanh(u);
    double s = smin(1.0 - tl * tl, 1.0 - tu * tu);
    *slope = s;
    double lo_int = tl - s * l, hi_int = lo_int;
    double g = tu - s * u;
    lo_int = smin(lo_int, g); hi_int = smax(hi_int, g);
    if (s < 1.0 && s > 0.0) {
      double xs = atanh(sqrt(1.0 - s));
      if (l <= xs && xs <= u) { g = tanh(xs) - s * xs; lo_int = smin(lo_int, g); hi_int = smax(hi_int, g); }
      if (l <= -xs && -xs <= u) { g = tanh(-xs) - s * -xs; lo_int = smin(lo_int, g); hi_int = smax(hi_int, g); }
    }
    double margin = (hi_int - lo_int) * 1e-12 + 1e-15;
    *li = lo_int - margin;
    *ui = hi_int + margin;
  }
  return 0;
}

/* act_interval (neural.hpp:229-241). */
static iv act_interval(int act, iv p) {
  iv r = p;
  if (act == REACH_ACT_RELU) { r.lo = smax(p.lo, 0.0); r.hi = smax(p.hi, 0.0); }
  else if (act == REACH_ACT_TANH) { r.lo = tanh(p.lo); r.hi = tanh(p.hi); }
  return r;
}

/*
 * certify_tm_input (neural.hpp:342-394) on the prepended wide network,
 * with crown_backward (neural.hpp:290-335) and preactivation_bounds
 * (neural.hpp:243-257) inlined.  Input TM: x = c + A z + r, z in [-1,1]^nz,
 * r in ig (time_horizon = 0).  `net` layers 0..L-1 are the (frozen) network;
 * layer 0 of `net` has n_i columns.  Outputs: out_c[n_o], out_A[n_o x nz]
 * (ld nz), rem[n_o].  Returns 0 ok, 1 non-finite preactivation.
 */
static int certify_tm_input(const net_t* net, int n_i, int nz, const double* c, const double* A /* n_i x nz */,
                            const iv* ig, double* out_c, double* out_A, iv* rem) {
  const int L = net->n_layers;
  const int n_o = net->layers[L - 1].rows;
  const int wcols = nz + n_i;
  int maxw = wcols;
  for (int l = 0; l < L; ++l) { if (net->layers[l].rows > maxw) maxw = net->layers[l].rows; if (net->layers[l].cols > maxw) maxw = net->layers[l].cols; }
  /* preactivation boxes: wide layer 0 (prepend) then net layers */
  iv** pre = (iv**)malloc(sizeof(iv*) * (size_t)(L + 1));
  pre[0] = (iv*)malloc(sizeof(iv) * (size_t)n_i);
  for (int l = 0; l < L; ++l) pre[l + 1] = (iv*)malloc(sizeof(iv) * (size_t)net->layers[l].rows);
  iv* h = (iv*)malloc(sizeof(iv) * (size_t)maxw);
  iv* hn = (iv*)malloc(sizeof(iv) * (size_t)maxw);
  /* prepend layer: W = [A | I], b = c, domain [-1,1]^nz x ig (neural.hpp:360-373),
     box_affine_image (interval.hpp:284-295) */
  for (int i = 0; i < n_i; ++i) {
    iv acc = {0.0, 0.0};
    const iv unit = {-1.0, 1.0};
    for (int j = 0; j < nz; ++j) acc = iv_add(acc, iv_scale(A[(size_t)i * nz + j], unit));
    for (int j = 0; j < n_i; ++j) acc = iv_add(acc, iv_scale(j == i ? 1.0 : 0.0, ig[j]));
    iv bb = {c[i], c[i]};
    pre[0][i] = iv_add(acc, bb);
    h[i] = pre[0][i]; /* identity act */
  }
  int hw = n_i;
  for (int l = 0; l < L; ++l) {
    const layer_t* Ly = &net->layers[l];
    for (int i = 0; i < Ly->rows; ++i) {
      iv acc = {0.0, 0.0};
      for (int j = 0; j < Ly->cols; ++j) acc = iv_add(acc, iv_scale(Ly->w[(size_t)i * Ly->cols + j], h[j]));
      iv bb = {Ly->b[i], Ly->b[i]};
      pre[l + 1][i] = iv_add(acc, bb);
      hn[i] = act_interval(Ly->act, pre[l + 1][i]);
    }
    iv* t = h; h = hn; hn = t;
    hw = Ly->rows;
  }
  (void)hw;

  /* backward (neural.hpp:297-327), a = Lambda (n_o x width) row-major */
  double* a = (double*)malloc(sizeof(double) * (size_t)n_o * (size_t)(maxw > n_o ? maxw : n_o));
  double* an = (double*)malloc(sizeof(double) * (size_t)n_o * (size_t)(maxw > n_o ? maxw : n_o));
  double* b_lo = (double*)calloc((size_t)n_o, sizeof(double));
  double* b_up = (double*)calloc((size_t)n_o, sizeof(double));
  double* shift = (double*)malloc(sizeof(double) * (size_t)n_o);
  int acols = n_o;
  for (int i = 0; i < n_o; ++i)
    for (int j = 0; j < n_o; ++j) a[(size_t)i * n_o + j] = (i == j) ? 1.0 : 0.0;
  int status = 0;
  for (int l = L; l >= 0 && status == 0; --l) {
    /* wide layer l: l == 0 is the prepend layer, else net layer l-1 */
    int rows, cols, act;
    const double* w = NULL; const double* bias = NULL;
    if (l == 0) { rows = n_i; cols = wcols; act = REACH_ACT_IDENTITY; bias = c; }
    else { const layer_t* Ly = &net->layers[l - 1]; rows = Ly->rows; cols = Ly->cols; act = Ly->act; w = Ly->w; bias = Ly->b; }
    (void)rows;
    if (act != REACH_ACT_IDENTITY) {
      for (int j = 0; j < acols; ++j) {
        double s, li, ui;
        if (relax_activation(act, pre[l][j], &s, &li, &ui)) { status = 1; break; }
        for (int i = 0; i < n_o; ++i) {
          double aij = a[(size_t)i * acols + j];
          if (aij >= 0.0) { b_lo[i] += aij * li; b_up[i] += aij * ui; }
          else { b_lo[i] += aij * ui; b_up[i] += aij * li; }
          a[(size_t)i * acols + j] = aij * s;
        }
      }
      if (status) break;
    }
    /* shift = matvec(a, b) (linalg.hpp:40-51); b += shift (vadd) */
    for (int i = 0; i < n_o; ++i) {
      double acc = 0.0;
      for (int j = 0; j < acols; ++j) acc += a[(size_t)i * acols + j] * bias[j];
      shift[i] = acc;
    }
    for (int i = 0; i < n_o; ++i) { b_lo[i] = b_lo[i] + shift[i]; b_up[i] = b_up[i] + shift[i]; }
    /* a = matmul(a, W) (linalg.hpp:53-63), i-k-j order */
    for (int i = 0; i < n_o; ++i) {
      double* crow = an + (size_t)i * cols;
      for (int j = 0; j < cols; ++j) crow[j] = 0.0;
      for (int k = 0; k < acols; ++k) {
        double aik = a[(size_t)i * acols + k];
        if (l == 0) {
          for (int j = 0; j < nz; ++j) crow[j] += aik * A[(size_t)k * nz + j];
          for (int j = 0; j < n_i; ++j) crow[nz + j] += aik * ((j == k) ? 1.0 : 0.0);
        } else {
          const double* wrow = w + (size_t)k * cols;
          for (int j = 0; j < cols; ++j) crow[j] += aik * wrow[j];
        }
      }
    }
    double* t = a; a = an; an = t;
    acols = cols;
  }
  if (status == 0) {
    /* tail (neural.hpp:383-391) */
    for (int i = 0; i < n_o; ++i) {
      double mid = (b_lo[i] + b_up[i]) * 0.5;
      out_c[i] = mid;
      for (int j = 0; j < nz; ++j) out_A[(size_t)i * nz + j] = a[(size_t)i * wcols + j];
      iv r = {b_lo[i] - mid, b_up[i] - mid};
      for (int j = 0; j < n_i; ++j) r = iv_add(r, iv_scale(a[(size_t)i * wcols + nz + j], ig[j]));
      rem[i] = r;
    }
  }
  for (int l = 0; l <= L; ++l) free(pre[l]);
  free(pre); free(h); free(hn); free(a); free(an); free(b_lo); free(b_up); free(shift);
  return status;
}

/* mat_solve (linalg.hpp:96-132): A X = B, A n x n, B n x m, partial pivoting. */
static int mat_solve(int n, int m, const double* A0, const double* B0, double* X) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* b = (double*)malloc(sizeof(double) * (size_t)n * m);
  memcpy(a, A0, sizeof(double) * (size_t)n * n);
  memcpy(b, B0, sizeof(double) * (size_t)n * m);
  int ok = 1;
  for (int k = 0; k < n && ok; ++k) {
    int piv = k;
    double best = fabs(a[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double cand = fabs(a[(size_t)i * n + k]);
      if (cand > best) { best = cand; piv = i; }
    }
    if (!(best > 1e-12)) { ok = 0; break; }
    if (piv != k) {
      for (int j = 0; j < n; ++j) { double t = a[(size_t)k * n + j]; a[(size_t)k * n + j] = a[(size_t)piv * n + j]; a[(size_t)piv * n + j] = t; }
      for (int j = 0; j < m; ++j) { double t = b[(size_t)k * m + j]; b[(size_t)k * m + j] = b[(size_t)piv * m + j]; b[(size_t)piv * m + j] = t; }
    }
    for (int i = k + 1; i < n; ++i) {
      double f = a[(size_t)i * n + k] / a[(size_t)k * n + k];
      for (int j = k; j < n; ++j) a[(size_t)i * n + j] -= f * a[(size_t)k * n + j];
      for (int j = 0; j < m; ++j) b[(size_t)i * m + j] -= f * b[(size_t)k * m + j];
    }
  }
  if (ok) {
    for (int i = n - 1; i >= 0; --i)
      for (int j = 0; j < m; ++j) {
        double acc = b[(size_t)i * m + j];
        for (int k = i + 1; k < n; ++k) acc -= a[(size_t)i * n + k] * X[(size_t)k * m + j];
        X[(size_t)i * m + j] = acc / a[(size_t)i * n + i];
      }
  }
  free(a); free(b);
  return ok;
}

static double row_abs_sum(const double* M, int cols, int i) {
  double acc = 0.0;
  for (int j = 0; j < cols; ++j) acc += fabs(M[(size_t)i * cols + j]);
  return acc;
}

/* SymbolicState (flowpipe_ct.hpp:286-300) for the DT path: every block is
 * n x n (G0 from the diagonal init, fresh blocks n x n). blocks[0] = G0,
 * blocks[1..nq] = queue oldest..newest. */
typedef struct {
  int n, nq, window;
  double* c;      /* n */
  double* blocks; /* (window+3) * n * n */
} symstate;

static int sym_cap(const symstate* s) { return s->window > 0 ? s->window : 1; }
static double* blk(symstate* s, int b) { return s->blocks + (size_t)b * s->n * s->n; }

/* init_symbolic_state (flowpipe_ct.hpp:303-309) */
static void sym_init(symstate* s, const double* lo, const double* hi) {
  const int n = s->n;
  s->nq = 0;
  double* g0 = blk(s, 0);
  memset(g0, 0, sizeof(double) * (size_t)n * n);
  for (int i = 0; i < n; ++i) {
    s->c[i] = (lo[i] + hi[i]) * 0.5;          /* Interval::mid */
    g0[(size_t)i * n + i] = (hi[i] - lo[i]) * 0.5; /* Interval::rad */
  }
}

/* fold_overflow (flowpipe_ct.hpp:317-350) */
static void fold_overflow(symstate* s) {
  const int n = s->n;
  double* x = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* e = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  while (s->nq > sym_cap(s)) {
    double* a = blk(s, 1);
    double* newest = blk(s, s->nq);
    double* g0 = blk(s, 0);
    int folded = 0;
    if (mat_solve(n, n, g0, a, x)) {
      double worst = 0.0;
      for (int j = 0; j < n; ++j) {
        r[j] = row_abs_sum(x, n, j) * (1.0 + 1e-12);
        worst = smax(worst, r[j]); /* std::max(worst, value(r_j)) */
      }
      if (worst <= 1.0) {
        for (int i = 0; i < n; ++i) {
          for (int j = 0; j < n; ++j) e[(size_t)i * n + j] = 0.0;
          for (int k = 0; k < n; ++k) {
            double gik = g0[(size_t)i * n + k];
            for (int j = 0; j < n; ++j) e[(size_t)i * n + j] += gik * x[(size_t)k * n + j];
          }
        }
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) e[(size_t)i * n + j] -= a[(size_t)i * n + j];
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) g0[(size_t)i * n + j] *= 1.0 + r[j];
        for (int i = 0; i < n; ++i) newest[(size_t)i * n + i] += row_abs_sum(e, n, i) * (1.0 + 1e-12);
        folded = 1;
      }
    }
    if (!folded)
      for (int i = 0; i < n; ++i) newest[(size_t)i * n + i] += row_abs_sum(a, n, i);
    /* pop_front */
    memmove(blk(s, 1), blk(s, 2), sizeof(double) * (size_t)n * n * (size_t)(s->nq - 1));
    s->nq -= 1;
  }
  free(x); free(e); free(r);
}

/*
 * dt_reach (dt_reach.hpp:41-104) for one sample.  Writes boxes into lo/hi
 * ([H+1][n]); returns n_boxes; *failed_step / *status per tube.hpp:30-34.
 */
static int dt_reach_one(const net_t* net, int n, int m, int H, int window, int rebuild,
                        const double* x0lo, const double* x0hi, const double* actions,
                        double* lo, double* hi, int* failed_step, int* status) {
  const int cap = window > 0 ? window : 1;
  const int nzmax = n * (cap + 2);
  symstate s;
  s.n = n; s.window = window; s.nq = 0;
  s.c = (double*)malloc(sizeof(double) * (size_t)n);
  s.blocks = (double*)calloc((size_t)(cap + 3) * n * n, sizeof(double));
  double* A = (double*)malloc(sizeof(double) * (size_t)n * nzmax);
  double* oc = (double*)malloc(sizeof(double) * (size_t)n);
  double* oA = (double*)malloc(sizeof(double) * (size_t)n * nzmax);
  iv* rem = (iv*)malloc(sizeof(iv) * (size_t)n);
  iv* ig = (iv*)calloc((size_t)n, sizeof(iv));
  double* bias = NULL;
  /* frozen network copy (freeze_trailing_inputs, neural.hpp:398-413) */
  net_t fz = *net;
  fz.layers = (layer_t*)malloc(sizeof(layer_t) * (size_t)net->n_layers);
  memcpy(fz.layers, net->layers, sizeof(layer_t) * (size_t)net->n_layers);
  const layer_t* l0 = &net->layers[0];
  double* w0 = NULL;
  if (m > 0) {
    w0 = (double*)malloc(sizeof(double) * (size_t)l0->rows * n);
    for (int i = 0; i < l0->rows; ++i)
      for (int j = 0; j < n; ++j) w0[(size_t)i * n + j] = l0->w[(size_t)i * l0->cols + j];
    bias = (double*)malloc(sizeof(double) * (size_t)l0->rows);
    fz.layers[0].w = w0;
    fz.layers[0].cols = n;
    fz.layers[0].b = bias;
  }

  int nb = 0;
  *failed_step = -1;
  *status = REACH_TUBE_OK;
  for (int d = 0; d < n; ++d) { lo[d] = x0lo[d]; hi[d] = x0hi[d]; }
  nb = 1;
  sym_init(&s, x0lo, x0hi);
  for (int k = 0; k < H; ++k) {
    if (m > 0) {
      const double* u = actions + (size_t)k * m;
      for (int i = 0; i < l0->rows; ++i) {
        double bi = l0->b[i];
        for (int j = 0; j < m; ++j) bi += l0->w[(size_t)i * l0->cols + n + j] * u[j];
        bias[i] = bi;
      }
    }
    /* symbolic_seed (flowpipe_ct.hpp:353-370): A = [G0 | Q1 .. Qk] */
    const int nz = n * (1 + s.nq);
    for (int i = 0; i < n; ++i)
      for (int b = 0; b <= s.nq; ++b)
        for (int j = 0; j < n; ++j) A[(size_t)i * nz + b * n + j] = blk(&s, b)[(size_t)i * n + j];
    if (certify_tm_input(&fz, n, nz, s.c, A, ig, oc, oA, rem)) {
      *failed_step = k; *status = REACH_TUBE_NONFINITE_PREACT; break;
    }
    int fin = 1;
    for (int i = 0; i < n; ++i) if (!iv_finite(rem[i])) fin = 0;
    if (!fin) { *failed_step = k; *status = REACH_TUBE_DIVERGED_CERT; break; }
    /* re-seed (dt_reach.hpp:69-92) */
    for (int i = 0; i < n; ++i) s.c[i] = oc[i] + (rem[i].lo + rem[i].hi) * 0.5;
    for (int b = 0; b <= s.nq; ++b)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) blk(&s, b)[(size_t)i * n + j] = oA[(size_t)i * nz + b * n + j];
    s.nq += 1;
    double* fresh = blk(&s, s.nq);
    memset(fresh, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) fresh[(size_t)i * n + i] = (rem[i].hi - rem[i].lo) * 0.5;
    fold_overflow(&s);
    /* symbolic_box (flowpipe_ct.hpp:413-424) */
    int bfin = 1;
    double* blo = lo + (size_t)nb * n;
    double* bhi = hi + (size_t)nb * n;
    for (int i = 0; i < n; ++i) {
      double r = row_abs_sum(blk(&s, 0), n, i);
      for (int b = 1; b <= s.nq; ++b) r += row_abs_sum(blk(&s, b), n, i);
      blo[i] = s.c[i] - r;
      bhi[i] = s.c[i] + r;
      if (!isfinite(blo[i]) || !isfinite(bhi[i])) bfin = 0;
    }
    nb += 1;
    if (!bfin) { *failed_step = k; *status = REACH_TUBE_DIVERGED_BOX; break; }
    if (rebuild) sym_init(&s, blo, bhi);
  }
  free(s.c); free(s.blocks); free(A); free(oc); free(oA); free(rem); free(ig);
  free(fz.layers); free(w0); free(bias);
  return nb;
}

int orc_dt_batch(const reach_net_desc* desc, const reach_dt_args* a, const reach_tube_out* out) {
  if (!desc || !a || !out || a->n <= 0 || a->m < 0 || a->horizon < 0 || a->batch < 0) return REACH_E_INVALID_ARGUMENT;
  if (desc->dims[0] != a->n + a->m || desc->dims[desc->n_layers] != a->n) return REACH_E_INVALID_ARGUMENT;
  net_t net = net_from_desc(desc);
  const int H = a->horizon, n = a->n, m = a->m;
  for (int b = 0; b < a->batch; ++b) {
    const double* act = a->actions_shared ? a->actions : a->actions + (size_t)b * H * m;
    int fs, st;
    int nb = dt_reach_one(&net, n, m, H, a->window, a->rebuild_from_box, a->x0_lo + (size_t)b * n,
                          a->x0_hi + (size_t)b * n, act, out->lo + (size_t)b * (H + 1) * n,
                          out->hi + (size_t)b * (H + 1) * n, &fs, &st);
    out->n_boxes[b] = nb;
    out->failed_step[b] = fs;
    out->status[b] = st;
  }
  free(net.layers);
  return REACH_OK;
}

/* split_box (refine.hpp:83-115) part p (last dim fastest) into lo/hi. */
static void split_part(int n, const double* xlo, const double* xhi, const int32_t* counts, int64_t p,
                       double* lo, double* hi) {
  for (int d = n - 1; d >= 0; --d) {
    int k = counts[d];
    int i = (int)(p % k);
    p /= k;
    double e0 = (i == 0) ? xlo[d] : xlo[d] + (xhi[d] - xlo[d]) * ((double)i / k);
    double e1 = (i + 1 == k) ? xhi[d] : xlo[d] + (xhi[d] - xlo[d]) * ((double)(i + 1) / k);
    lo[d] = e0;
    hi[d] = e1;
  }
}

/* reach_with_splitting hull reduction (refine.hpp:133-158) over parts [begin,end). */
int orc_split_hull(const reach_net_desc* desc, const reach_split_args* a, const reach_hull_out* out) {
  const int n = a->n, H = a->horizon;
  int64_t total = 1;
  for (int d = 0; d < n; ++d) { if (a->counts[d] < 1) return REACH_E_INVALID_ARGUMENT; total *= a->counts[d]; }
  int64_t begin = a->part_begin, end = a->part_end <= 0 ? total : a->part_end;
  if (begin < 0 || begin >= end || end > total) return REACH_E_INVALID_ARGUMENT;
  net_t net = net_from_desc(desc);
  double* lo = (double*)malloc(sizeof(double) * (size_t)(H + 1) * n);
  double* hi = (double*)malloc(sizeof(double) * (size_t)(H + 1) * n);
  double plo[64], phi[64];
  int steps = 0;
  int64_t key = INT64_MAX;
  for (int64_t p = begin; p < end; ++p) {
    split_part(n, a->x0_lo, a->x0_hi, a->counts, p, plo, phi);
    int fs, st;
    int nb = dt_reach_one(&net, n, a->m, H, a->window, a->rebuild_from_box, plo, phi, a->actions, lo, hi, &fs, &st);
    if (p == begin) {
      steps = nb;
      for (int k = 0; k < nb; ++k) {
        for (int d = 0; d < n; ++d) { out->lo[k * n + d] = lo[k * n + d]; out->hi[k * n + d] = hi[k * n + d]; }
      }
      for (int k = 0; k <= H; ++k) out->box_diverged[k] = 0;
    } else {
      int upto = nb < steps ? nb : steps;
      for (int k = 0; k < upto; ++k)
        for (int d = 0; d < n; ++d) {
          out->lo[k * n + d] = smin(out->lo[k * n + d], lo[k * n + d]);
          out->hi[k * n + d] = smax(out->hi[k * n + d], hi[k * n + d]);
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
  free(lo); free(hi); free(net.layers);
  return REACH_OK;
}

/* ======================================================================= */
/* Reachability-aware MPC (mpc.hpp): plan_eval and plan_cem restated.       */

/* MLPNet::forward (neural.hpp:58-76): matvec then + b, ReLU as h_relu. */
static void mlp_forward(const net_t* net, const double* in, double* out, double* buf1, double* buf2) {
  const double* h = in;
  double* bufs[2] = {buf1, buf2};
  for (int l = 0; l < net->n_layers; ++l) {
    const layer_t* Ly = &net->layers[l];
    double* o = bufs[l & 1];
    for (int i = 0; i < Ly->rows; ++i) {
      double acc = 0.0;
      for (int j = 0; j < Ly->cols; ++j) acc += Ly->w[(size_t)i * Ly->cols + j] * h[j];
      double v = acc + Ly->b[i];
      if (Ly->act == REACH_ACT_RELU) { if (v < 0.0) v = 0.0; }
      else if (Ly->act == REACH_ACT_TANH) v = tanh(v);
      o[i] = v;
    }
    h = o;
  }
  memcpy(out, h, sizeof(double) * (size_t)net->layers[net->n_layers - 1].rows);
}

/* Constraint::margin (mpc.hpp:40-86). */
static double con_margin(const reach_constraint* c, int n, const double* lo, const double* hi) {
  const int k = c->n_dims > 0 ? c->n_dims : n;
  switch (c->type) {
    case REACH_CON_HALFSPACE_AVOID: {
      double worst = c->b;
      for (int j = 0; j < k; ++j) {
        const int d = c->n_dims > 0 ? c->dims[j] : j;
        const double term = c->a[j] >= 0.0 ? hi[d] * c->a[j] : lo[d] * c->a[j];
        worst -= term;
      }
      return worst;
    }
    case REACH_CON_SPHERE_AVOID: {
      double d2 = 0.0;
      for (int j = 0; j < k; ++j) {
        const int d = c->n_dims > 0 ? c->dims[j] : j;
        double gap = 0.0;
        if (lo[d] > c->center[j]) gap = lo[d] - c->center[j];
        else if (hi[d] < c->center[j]) gap = c->center[j] - hi[d];
        d2 += gap * gap;
      }
      return sqrt(d2) - c->radius;
    }
    case REACH_CON_BOX_STAY_IN: {
      double worst = INFINITY;
      for (int j = 0; j < k; ++j) {
        const int d = c->n_dims > 0 ? c->dims[j] : j;
        worst = smin(worst, lo[d] - c->lo[j]);
        worst = smin(worst, c->hi[j] - hi[d]);
      }
      return worst;
    }
    default: {
      double v = 0.0;
      for (int j = 0; j < k; ++j) {
        const int d = c->n_dims > 0 ? c->dims[j] : j;
        v += hi[d] - lo[d];
      }
      return c->vmax - v;
    }
  }
}

/* plan_eval (mpc.hpp:158-202) for one candidate. */
static double plan_eval_one(const net_t* net, const reach_plan_problem* p, const double* x0, const double* acts,
                            int* diverged) {
  const int n = p->n, m = p->m, H = p->horizon;
  int maxw = n + m;
  for (int l = 0; l < net->n_layers; ++l) if (net->layers[l].rows > maxw) maxw = net->layers[l].rows;
  double* x = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* in = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* b1 = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* b2 = (double*)malloc(sizeof(double) * (size_t)maxw);
  double obj = 0.0;
  memcpy(x, x0, sizeof(double) * (size_t)n);
  for (int t = 0; t < H; ++t) {
    const double* u = acts + (size_t)t * m;
    memcpy(in, x, sizeof(double) * (size_t)n);
    memcpy(in + n, u, sizeof(double) * (size_t)m);
    mlp_forward(net, in, x, b1, b2);
    for (int j = 0; j < m; ++j) obj += p->r_weights[j] * u[j] * u[j];
    for (int j = 0; j < n; ++j) {
      const double d = x[j] - p->x_goal[j];
      obj += p->q_weights[j] * d * d;
    }
  }
  /* tube at radius eps: box_from_center (interval.hpp:224-235) */
  double* lo0 = (double*)malloc(sizeof(double) * (size_t)n);
  double* hi0 = (double*)malloc(sizeof(double) * (size_t)n);
  for (int d = 0; d < n; ++d) { lo0[d] = x0[d] - p->eps; hi0[d] = x0[d] + p->eps; }
  double* tlo = (double*)malloc(sizeof(double) * (size_t)(H + 1) * n);
  double* thi = (double*)malloc(sizeof(double) * (size_t)(H + 1) * n);
  int fs, st;
  const int nb = dt_reach_one(net, n, m, H, p->window, p->rebuild_from_box, lo0, hi0, acts, tlo, thi, &fs, &st);
  *diverged = st != REACH_TUBE_OK;
  for (int t = 1; t <= H; ++t) {
    int ok = t < nb;
    for (int d = 0; ok && d < n; ++d)
      if (!isfinite(tlo[(size_t)t * n + d]) || !isfinite(thi[(size_t)t * n + d])) ok = 0;
    if (ok) {
      for (int c = 0; c < p->n_constraints; ++c) {
        const double g = con_margin(&p->constraints[c], n, tlo + (size_t)t * n, thi + (size_t)t * n);
        obj += p->penalty * smax(0.0, -g);
      }
    } else if (p->n_constraints > 0) {
      obj += p->penalty * p->diverged_margin * (double)p->n_constraints;
    }
  }
  free(x); free(in); free(b1); free(b2); free(lo0); free(hi0); free(tlo); free(thi);
  return obj;
}

int orc_plan_eval_batch(const reach_net_desc* desc, const reach_plan_problem* p, const double* x0, int32_t batch,
                        const double* actions, double* objective, int32_t* diverged) {
  net_t net = net_from_desc(desc);
  for (int b = 0; b < batch; ++b) {
    int dv;
    objective[b] = plan_eval_one(&net, p, x0, actions + (size_t)b * p->horizon * p->m, &dv);
    diverged[b] = dv;
  }
  free(net.layers);
  return REACH_OK;
}

/* std::mt19937_64 (the reference Rng's engine, rng.hpp:13-52). */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}
static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
typedef struct { mt64 g; int has_spare; double spare; } rng_t;
static double rng_u01(rng_t* r) { return (double)(mt64_next(&r->g) >> 11) * 0x1.0p-53; }
static double rng_normal(rng_t* r) { /* Rng::normal, cached Box-Muller */
  if (r->has_spare) { r->has_spare = 0; return r->spare; }
  double u1 = rng_u01(r), u2 = rng_u01(r);
  while (u1 <= 0.0) u1 = rng_u01(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double a = 6.28318530717958647692 * u2;
  r->spare = rad * sin(a);
  r->has_spare = 1;
  return rad * cos(a);
}
static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; } /* std::clamp */

static const double* g_sort_scores;
static int cmp_score_index(const void* a, const void* b) {  /* stable ascending: (score, index) */
  const int ia = *(const int*)a, ib = *(const int*)b;
  const double sa = g_sort_scores[ia], sb = g_sort_scores[ib];
  if (sa < sb) return -1;
  if (sb < sa) return 1;
  return (ia > ib) - (ia < ib);
}

/* plan_cem (mpc.hpp:258-368) with refine_iters == 0 (single-threaded restatement). */
int orc_plan_cem(const reach_net_desc* desc, const reach_plan_problem* p, const reach_sampler_config* cfg,
                 const double* x0, double* best_actions, double* objective, double* best_history, int32_t* best_effort) {
  if (cfg->refine_iters != 0) return REACH_E_UNSUPPORTED;
  net_t net = net_from_desc(desc);
  const int h = p->horizon, m = p->m, pop = cfg->population;
  const size_t dim = (size_t)h * m;
  rng_t rng; mt64_seed(&rng.g, cfg->seed); rng.has_spare = 0; rng.spare = 0.0;
  double* mean = (double*)malloc(sizeof(double) * dim);
  double* stdv = (double*)malloc(sizeof(double) * dim);
  double* best = (double*)malloc(sizeof(double) * dim);
  double* cands = (double*)malloc(sizeof(double) * dim * (size_t)pop);
  double* scores = (double*)malloc(sizeof(double) * (size_t)pop);
  int* okv = (int*)malloc(sizeof(int) * (size_t)pop);
  int* order = (int*)malloc(sizeof(int) * (size_t)pop);
  for (int t = 0; t < h; ++t)
    for (int j = 0; j < m; ++j) mean[(size_t)t * m + j] = 0.5 * (p->u_lo[j] + p->u_hi[j]);
  for (size_t k = 0; k < dim; ++k) { stdv[k] = cfg->init_std; best[k] = clampd(mean[k], p->u_lo[k % m], p->u_hi[k % m]); }
  double best_obj = INFINITY;
  int any_finite = 0;
  int n_elite = (int)(pop * cfg->elite_frac);
  if (n_elite < 1) n_elite = 1;
  for (int it = 0; it < cfg->iterations; ++it) {
    for (int c = 0; c < pop; ++c) {
      double* u = cands + (size_t)c * dim;
      if (it > 0 && c == 0) {
        memcpy(u, best, sizeof(double) * dim);
      } else {
        for (size_t k = 0; k < dim; ++k) u[k] = mean[k] + stdv[k] * rng_normal(&rng);
        for (size_t k = 0; k < dim; ++k) u[k] = clampd(u[k], p->u_lo[k % m], p->u_hi[k % m]);
      }
    }
    for (int c = 0; c < pop; ++c) {
      int dv;
      scores[c] = plan_eval_one(&net, p, x0, cands + (size_t)c * dim, &dv);
      okv[c] = !dv;
    }
    for (int c = 0; c < pop; ++c) order[c] = c;
    g_sort_scores = scores;
    qsort(order, (size_t)pop, sizeof(int), cmp_score_index);
    const int top = order[0];
    if (scores[top] < best_obj) { best_obj = scores[top]; memcpy(best, cands + (size_t)top * dim, sizeof(double) * dim); }
    for (int e = 0; e < n_elite; ++e) if (okv[order[e]]) any_finite = 1;
    best_history[it] = best_obj;
    for (size_t k = 0; k < dim; ++k) {
      double em = 0.0, ev = 0.0;
      for (int e = 0; e < n_elite; ++e) em += cands[(size_t)order[e] * dim + k];
      em /= n_elite;
      for (int e = 0; e < n_elite; ++e) { const double d = cands[(size_t)order[e] * dim + k] - em; ev += d * d; }
      const double es = sqrt(ev / n_elite);
      mean[k] = cfg->smoothing * mean[k] + (1.0 - cfg->smoothing) * em;
      stdv[k] = smax(1e-6, cfg->smoothing * stdv[k] + (1.0 - cfg->smoothing) * es);
    }
  }
  *best_effort = !any_finite;
  memcpy(best_actions, best, sizeof(double) * dim);
  int dv;
  *objective = plan_eval_one(&net, p, x0, best, &dv);
  free(mean); free(stdv); free(best); free(cands); free(scores); free(okv); free(order); free(net.layers);
  return REACH_OK;
}

/* ======================================================================= */
/* DT closed loop: the composition of reference        */
/* functions mirroring cl_reach's stacking (closed_loop.hpp:118-153), with */
/* generator blocks of varying widths.                                      */

typedef struct {
  int n, nq, window, ld;
  double* c;   /* n */
  double* S;   /* n x ld: [G0 | Q1 .. Qnq] */
  int* wid;    /* block widths */
} symv;

static int symv_nz(const symv* s) { int z = s->n; for (int q = 0; q < s->nq; ++q) z += s->wid[q]; return z; }

/* fold_overflow (flowpipe_ct.hpp:317-350) with an n x w oldest block. */
static void symv_fold(symv* s) {
  const int n = s->n, cap = s->window > 0 ? s->window : 1;
  while (s->nq > cap) {
    const int w = s->wid[0];
    double* g0 = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* a = (double*)malloc(sizeof(double) * (size_t)n * w);
    double* x = (double*)malloc(sizeof(double) * (size_t)n * w);
    double* e = (double*)malloc(sizeof(double) * (size_t)n * w);
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j) g0[(size_t)i * n + j] = s->S[(size_t)i * s->ld + j];
      for (int j = 0; j < w; ++j) a[(size_t)i * w + j] = s->S[(size_t)i * s->ld + n + j];
    }
    int off_new = n;
    for (int q = 0; q + 1 < s->nq; ++q) off_new += s->wid[q];
    int folded = 0;
    if (mat_solve(n, w, g0, a, x)) {
      double worst = 0.0;
      for (int j = 0; j < n; ++j) {
        r[j] = row_abs_sum(x, w, j) * (1.0 + 1e-12);
        worst = smax(worst, r[j]);
      }
      if (worst <= 1.0) {
        for (int i = 0; i < n; ++i) {
          for (int j = 0; j < w; ++j) e[(size_t)i * w + j] = 0.0;
          for (int k = 0; k < n; ++k) {
            const double gik = g0[(size_t)i * n + k];
            for (int j = 0; j < w; ++j) e[(size_t)i * w + j] += gik * x[(size_t)k * w + j];
          }
        }
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < w; ++j) e[(size_t)i * w + j] -= a[(size_t)i * w + j];
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i) s->S[(size_t)i * s->ld + j] *= 1.0 + r[j];
        for (int i = 0; i < n; ++i) s->S[(size_t)i * s->ld + off_new + i] += row_abs_sum(e, w, i) * (1.0 + 1e-12);
        folded = 1;
      }
    }
    if (!folded)
      for (int i = 0; i < n; ++i) s->S[(size_t)i * s->ld + off_new + i] += row_abs_sum(a, w, i);
    const int total = symv_nz(s);
    for (int i = 0; i < n; ++i)
      memmove(s->S + (size_t)i * s->ld + n, s->S + (size_t)i * s->ld + n + w, sizeof(double) * (size_t)(total - n - w));
    memmove(s->wid, s->wid + 1, sizeof(int) * (size_t)(s->nq - 1));
    s->nq -= 1;
    free(g0); free(a); free(x); free(e); free(r);
  }
}

static int dtcl_one(const net_t* dyn, const net_t* ctl, int n, int H, int window, int rebuild, const double* x0lo,
                    const double* x0hi, double* lo, double* hi, int* failed_step, int* status) {
  const int l = ctl->layers[ctl->n_layers - 1].rows;
  const int cap = window > 0 ? window : 1;
  const int ld = n + (cap + 3) * (n + l);
  symv s;
  s.n = n; s.nq = 0; s.window = window; s.ld = ld;
  s.c = (double*)malloc(sizeof(double) * (size_t)n);
  s.S = (double*)calloc((size_t)n * ld, sizeof(double));
  s.wid = (int*)malloc(sizeof(int) * (size_t)(cap + 4));
  double* A = (double*)malloc(sizeof(double) * (size_t)(n + l) * ld);
  double* uc = (double*)malloc(sizeof(double) * (size_t)l);
  double* uA = (double*)malloc(sizeof(double) * (size_t)l * ld);
  iv* urem = (iv*)malloc(sizeof(iv) * (size_t)l);
  double* cag = (double*)malloc(sizeof(double) * (size_t)(n + l));
  double* oc = (double*)malloc(sizeof(double) * (size_t)n);
  double* oA = (double*)malloc(sizeof(double) * (size_t)n * ld);
  iv* rem = (iv*)malloc(sizeof(iv) * (size_t)n);
  iv* ig = (iv*)calloc((size_t)(n + l), sizeof(iv));
  *failed_step = -1;
  *status = REACH_TUBE_OK;
  for (int d = 0; d < n; ++d) { lo[d] = x0lo[d]; hi[d] = x0hi[d]; }
  int nb = 1;
  /* init_symbolic_state */
  for (int i = 0; i < n; ++i) {
    s.c[i] = (x0lo[i] + x0hi[i]) * 0.5;
    for (int j = 0; j < n; ++j) s.S[(size_t)i * ld + j] = (i == j) ? (x0hi[i] - x0lo[i]) * 0.5 : 0.0;
  }
  for (int k = 0; k < H; ++k) {
    const int nz = symv_nz(&s);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < nz; ++j) A[(size_t)i * nz + j] = s.S[(size_t)i * ld + j];
    /* u_tm = ctl_crown(x_tm, ctl, {}) */
    if (certify_tm_input(ctl, n, nz, s.c, A, ig, uc, uA, urem)) { *failed_step = k; *status = REACH_TUBE_CTL_FAILED; break; }
    int fin = 1;
    for (int i = 0; i < l; ++i) if (!iv_finite(urem[i])) fin = 0;
    if (!fin) { *failed_step = k; *status = REACH_TUBE_CTL_DIVERGED; break; }
    /* stacked [x; u] over nz + (n + l) variables */
    const int w_new = n + l, nza = nz + w_new;
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < nza; ++j) A[(size_t)i * nza + j] = (j < nz) ? s.S[(size_t)i * ld + j] : 0.0;
      cag[i] = s.c[i] + (0.0 + 0.0) * 0.5;
    }
    for (int i = 0; i < l; ++i) {
      for (int j = 0; j < nza; ++j)
        A[(size_t)(n + i) * nza + j] = (j < nz) ? uA[(size_t)i * nz + j] : ((j - nz == n + i) ? (urem[i].hi - urem[i].lo) * 0.5 : 0.0);
      cag[n + i] = uc[i] + (urem[i].lo + urem[i].hi) * 0.5;
    }
    if (certify_tm_input(dyn, n + l, nza, cag, A, ig, oc, oA, rem)) { *failed_step = k; *status = REACH_TUBE_NONFINITE_PREACT; break; }
    for (int i = 0; i < n; ++i) if (!iv_finite(rem[i])) fin = 0;
    if (!fin) { *failed_step = k; *status = REACH_TUBE_DIVERGED_CERT; break; }
    for (int i = 0; i < n; ++i) {
      s.c[i] = oc[i] + (rem[i].lo + rem[i].hi) * 0.5;
      for (int j = 0; j < nza; ++j) s.S[(size_t)i * ld + j] = oA[(size_t)i * nza + j];
      for (int j = 0; j < n; ++j) s.S[(size_t)i * ld + nza + j] = (i == j) ? (rem[i].hi - rem[i].lo) * 0.5 : 0.0;
    }
    s.wid[s.nq++] = w_new;
    s.wid[s.nq++] = n;
    symv_fold(&s);
    /* symbolic_box */
    int bfin = 1;
    double* blo = lo + (size_t)nb * n;
    double* bhi = hi + (size_t)nb * n;
    for (int i = 0; i < n; ++i) {
      double r = row_abs_sum(s.S + (size_t)i * ld, n, 0);
      int off = n;
      for (int q = 0; q < s.nq; ++q) { r += row_abs_sum(s.S + (size_t)i * ld + off, s.wid[q], 0); off += s.wid[q]; }
      blo[i] = s.c[i] - r;
      bhi[i] = s.c[i] + r;
      if (!isfinite(blo[i]) || !isfinite(bhi[i])) bfin = 0;
    }
    nb += 1;
    if (!bfin) { *failed_step = k; *status = REACH_TUBE_DIVERGED_BOX; break; }
    if (rebuild) {
      s.nq = 0;
      for (int i = 0; i < n; ++i) {
        s.c[i] = (blo[i] + bhi[i]) * 0.5;
        for (int j = 0; j < n; ++j) s.S[(size_t)i * ld + j] = (i == j) ? (bhi[i] - blo[i]) * 0.5 : 0.0;
      }
    }
  }
  free(s.c); free(s.S); free(s.wid); free(A); free(uc); free(uA); free(urem); free(cag); free(oc); free(oA);
  free(rem); free(ig);
  return nb;
}

int orc_dtcl_batch(const reach_net_desc* dyn_desc, const reach_net_desc* ctl_desc, const reach_dt_args* a,
                   const reach_tube_out* out) {
  net_t dyn = net_from_desc(dyn_desc), ctl = net_from_desc(ctl_desc);
  const int H = a->horizon, n = a->n;
  for (int b = 0; b < a->batch; ++b) {
    int fs, st;
    const int nb = dtcl_one(&dyn, &ctl, n, H, a->window, a->rebuild_from_box, a->x0_lo + (size_t)b * n,
                            a->x0_hi + (size_t)b * n, out->lo + (size_t)b * (H + 1) * n,
                            out->hi + (size_t)b * (H + 1) * n, &fs, &st);
    out->n_boxes[b] = nb;
    out->failed_step[b] = fs;
    out->status[b] = st;
  }
  free(dyn.layers); free(ctl.layers);
  return REACH_OK;
}

/* Bridges for ct_oracle.c. */
int orc_i_mat_solve(int n, int m, const double* A, const double* B, double* X) { return mat_solve(n, m, A, B, X); }
net_t orc_i_net_from_desc(const reach_net_desc* d) { return net_from_desc(d); }
int orc_i_certify_tm_input(const net_t* net, int n_i, int nz, const double* c, const double* A, const iv* ig,
                           double* out_c, double* out_A, iv* rem) {
  return certify_tm_input(net, n_i, nz, c, A, ig, out_c, out_A, rem);
}
