// Forward-mode dual gradients of the MPC planning objective on the device:
// grad_forward (refine.hpp:186-207) of plan_objective (mpc.hpp:158-208) over
// the flat action sequence, the gradient plan_cem's top-candidate refinement
// consumes (mpc.hpp:337-361, gradient_refine refine.hpp:347-398).
//
// One CTA per tangent direction j (action t = j / m, component j % m), all
// directions in one launch: each CTA evaluates the whole objective -- nominal
// rollout, dt_reach with certify_tm_input / crown_backward / fold_overflow /
// symbolic_box, constraint penalties -- in reach::Dual arithmetic
// (scalar.hpp:13-55) seeded with d(action_j) = 1, its working set (~120 KB)
// in shared memory.  Inside a CTA every output element of a layer (IBP row,
// Lambda.W entry, intercept row) is owned by one thread and accumulated in the
// reference's order with separate roundings, so ReLU networks give the
// reference's gradient bit for bit; reach::min / max / abs keep their Dual tie
// and NaN rules (a.v <= b.v ? a : b, ...).  Every branch of the reference's
// Dual pass depends on primal values only, so the CTAs follow one control path.
#pragma once

#include "dt_common.cuh"
#include "dt_kernel.cuh"
#include "plan.cuh"

namespace rb {
namespace dual {

constexpr int kN = 8;     // state dim
constexpr int kM = 4;     // action dim
constexpr int kW = 128;   // widest layer (and nz + n of the prepended layer)
constexpr int kL = 6;     // layers
constexpr int kZ = 80;    // generator columns incl. the fresh block
constexpr int kH = 64;    // horizon
constexpr int kQ = 12;    // queue blocks

// ---- reach::Dual (scalar.hpp:13-55) ------------------------------------------
struct D {
  double v, d;
};
__device__ __forceinline__ D dc(double v) { return D{v, 0.0}; }
__device__ __forceinline__ D dadd(D a, D b) { return D{add(a.v, b.v), add(a.d, b.d)}; }
__device__ __forceinline__ D dsub(D a, D b) { return D{sub(a.v, b.v), sub(a.d, b.d)}; }
__device__ __forceinline__ D dneg(D a) { return D{-a.v, -a.d}; }
__device__ __forceinline__ D dmul(D a, D b) { return D{mul(a.v, b.v), add(mul(a.d, b.v), mul(a.v, b.d))}; }
__device__ __forceinline__ D ddiv(D a, D b) {
  return D{__ddiv_rn(a.v, b.v), __ddiv_rn(sub(mul(a.d, b.v), mul(a.v, b.d)), mul(b.v, b.v))};
}
__device__ __forceinline__ D dmin(D a, D b) { return a.v <= b.v ? a : b; }
__device__ __forceinline__ D dmax(D a, D b) { return a.v >= b.v ? a : b; }
__device__ __forceinline__ D dabs(D a) { return a.v < 0.0 ? D{-a.v, -a.d} : a; }
__device__ __forceinline__ D dtanh(D a) {
  const double t = tanh(a.v);
  return D{t, mul(sub(1.0, mul(t, t)), a.d)};
}
__device__ __forceinline__ D dsqrt(D a) {
  const double s = __dsqrt_rn(a.v);
  return D{s, a.v > 0.0 ? __ddiv_rn(a.d, mul(2.0, s)) : 0.0};
}
__device__ __forceinline__ bool dfin(D a) { return isfinite(a.v); }

// ---- Interval<Dual> (interval.hpp:60-94) ----------------------------------------
struct DI {
  D lo, hi;
};
__device__ __forceinline__ DI iadd(DI a, DI b) { return DI{dadd(a.lo, b.lo), dadd(a.hi, b.hi)}; }
__device__ __forceinline__ DI iscale(D a, DI x) {
  return a.v >= 0.0 ? DI{dmul(a, x.lo), dmul(a, x.hi)} : DI{dmul(a, x.hi), dmul(a, x.lo)};
}
__device__ __forceinline__ D imid(DI x) { return dmul(dadd(x.lo, x.hi), dc(0.5)); }
__device__ __forceinline__ D irad(DI x) { return dmul(dsub(x.hi, x.lo), dc(0.5)); }

struct GradArgs {
  PlanParams P;         // net, n, m, H, goal / weights / constraints staged on the device
  int window, rebuild;
  double eps;
  const double* base;   // [H*m] the action sequence the gradient is taken at
  double* grad;         // [H*m] d objective / d action_j
  double* value;        // [H*m] primal objective seen by direction j
};

// Per-direction working set, in shared memory (one CTA per direction).
struct Work {
  D acts[kH][kM];
  D c[kN];
  D S[kN][kZ];          // [G0 | Q1 .. Qnq]
  int wid[kQ];
  int nq, stop, bad, sub;
  DI pre[kL - 1][kW];   // preactivations of the hidden layers
  union {
    DI hb[2][kW];       // IBP boxes / nominal activations (.lo)
    D rel[3][kW];       // crown: relaxation (slope, lower, upper intercept) of the current layer
  };
  D lam[2][kN][kW];     // Lambda, double buffered
  D blo[kN], bup[kN], shift[kN], bf0[kW];
  D oc[kN];
  D oA[kN][kZ];
  DI orem[kN];
  D tlo[kH + 1][kN], thi[kH + 1][kN];
  D g0[kN][kN], qa[kN][kN], qx[kN][kN], qe[kN][kN], rr[kN];
  D obj;
};

constexpr int kThreads = 256;
// two CTAs (directions) per SM: 2 x (Work + 1 KB static + 1 KB reserved) <= 228 KB
static_assert(sizeof(Work) <= 112 * 1024, "dual working set must fit two CTAs per SM");

// The network as Dual values: every parameter is a constant except, for a
// weights-target pass (grad_tube_volume, refine.hpp:234-236), the seeded one
// (layer sl, row si, column sj; sj = -1: the bias), whose value is shifted by
// `delta` (finite differences) and whose tangent is `seed`.
struct NetView {
  const DevNet& N;
  int sl = -1, si = -1, sj = -2;
  double delta = 0.0, seed = 0.0;
  __device__ __forceinline__ D pick(double v, int l, int i, int j) const {
    if (l != sl || i != si || j != sj) return dc(v);
    return D{delta != 0.0 ? add(v, delta) : v, seed};
  }
  __device__ __forceinline__ D w(int l, int i, int j) const {
    return pick(N.blob[N.w_off[l] + static_cast<long long>(i) * N.ldw[l] + j], l, i, j);
  }
  // W_l^T copy of the hidden layers: consecutive rows i are consecutive addresses
  __device__ __forceinline__ D wt(int l, int i, int j) const {
    return pick(N.blob[N.wt_off[l] + static_cast<long long>(j) * N.ldt[l] + i], l, i, j);
  }
  __device__ __forceinline__ D b(int l, int i) const { return pick(N.blob[N.b_off[l] + i], l, i, -1); }
};

// relax_activation (neural.hpp:166-227) on a Dual preactivation; false = throw.
__device__ inline bool relax_d(int act, DI pre, D& s, D& li, D& ui, bool& boundary) {
  if (!(dfin(pre.lo) && dfin(pre.hi))) return false;
  const D l = pre.lo, u = pre.hi;
  // note_branch_boundary (neural.hpp:180): the gradient is only a subgradient
  if (act == REACH_ACT_RELU && (l.v == 0.0 || u.v == 0.0)) boundary = true;
  s = dc(0.0);
  li = dc(0.0);
  ui = dc(0.0);
  if (act == REACH_ACT_IDENTITY) {
    s = dc(1.0);
  } else if (act == REACH_ACT_RELU) {
    if (l.v >= 0.0) {
      s = dc(1.0);
    } else if (u.v <= 0.0) {
      s = dc(0.0);
    } else {
      const D sl = ddiv(u, dsub(u, l));
      s = sl;
      ui = dmul(dneg(sl), l);
      li = dmin(dc(0.0), dmin(dmul(dneg(sl), l), dsub(u, dmul(sl, u))));
    }
  } else {  // tanh
    const D tl = dtanh(l), tu = dtanh(u);
    const D sl = dmin(dsub(dc(1.0), dmul(tl, tl)), dsub(dc(1.0), dmul(tu, tu)));
    s = sl;
    D lo_int = dsub(dtanh(l), dmul(sl, l));
    D hi_int = lo_int;
    auto consider = [&](D x) {
      const D g = dsub(dtanh(x), dmul(sl, x));
      lo_int = dmin(lo_int, g);
      hi_int = dmax(hi_int, g);
    };
    consider(u);
    if (sl.v < 1.0 && sl.v > 0.0) {
      const double xs = atanh(sqrt(1.0 - sl.v));
      if (l.v <= xs && xs <= u.v) consider(dc(xs));
      if (l.v <= -xs && -xs <= u.v) consider(dc(-xs));
    }
    const D margin = dadd(dmul(dsub(hi_int, lo_int), dc(1e-12)), dc(1e-15));
    li = dsub(lo_int, margin);
    ui = dadd(hi_int, margin);
  }
  return true;
}

__device__ __forceinline__ DI act_d(int act, DI p) {
  if (act == REACH_ACT_RELU) return DI{dmax(p.lo, dc(0.0)), dmax(p.hi, dc(0.0))};
  if (act == REACH_ACT_TANH) return DI{dtanh(p.lo), dtanh(p.hi)};
  return p;
}

// certify_tm_input (neural.hpp:342-394) of the frozen network on x = c + A z
// (A = W.S[:, :nz], zero remainder), by the whole CTA: every output element is
// owned by one thread and accumulated in the reference's order.  Returns 1 on a
// non-finite preactivation (relax_activation throws).  Ends synchronized.
__device__ __forceinline__ int certify_d(const NetView& net, int n, int nz, Work& W, int tid) {
  const DevNet& N = net.N;
  const int L = N.L, n_o = N.dims[L];
  // prepended layer [A | I], b = c, domain [-1,1]^nz x [0,0]^n (box_affine_image)
  for (int i = tid; i < n; i += kThreads) {
    DI acc{dc(0.0), dc(0.0)};
    for (int j = 0; j < nz; ++j) acc = iadd(acc, iscale(W.S[i][j], DI{dc(-1.0), dc(1.0)}));
    for (int j = 0; j < n; ++j) acc = iadd(acc, iscale(dc(i == j ? 1.0 : 0.0), DI{dc(0.0), dc(0.0)}));
    acc = iadd(acc, DI{W.c[i], W.c[i]});
    W.hb[0][i] = acc;
  }
  if (tid == 0) W.bad = 0;
  __syncthreads();
  int cur = 0;
  for (int t = 0; t + 1 < L; ++t) {  // IBP through the hidden layers (W^T rows: coalesced)
    const int rows = N.dims[t + 1], cols = (t == 0) ? n : N.dims[t];
    for (int u = tid; u < rows; u += kThreads) {
      DI acc{dc(0.0), dc(0.0)};
      if (net.sl != t) {
        const double* wrow = net.N.blob + net.N.wt_off[t] + u;
        const int ld = net.N.ldt[t];
#pragma unroll 4
        for (int j = 0; j < cols; ++j) acc = iadd(acc, iscale(dc(wrow[static_cast<long long>(j) * ld]), W.hb[cur][j]));
      } else {
        for (int j = 0; j < cols; ++j) acc = iadd(acc, iscale(net.wt(t, u, j), W.hb[cur][j]));
      }
      const D bias = (t == 0) ? W.bf0[u] : net.b(t, u);
      acc = iadd(acc, DI{bias, bias});
      W.pre[t][u] = acc;
      W.hb[cur ^ 1][u] = act_d(N.acts[t], acc);
    }
    cur ^= 1;
    __syncthreads();
  }
  // crown_backward (neural.hpp:290-335): Lambda = I
  int lb = 0, acols = n_o;
  for (int e = tid; e < n_o * n_o; e += kThreads) {
    const int i = e / n_o, j = e % n_o;
    W.lam[lb][i][j] = dc(i == j ? 1.0 : 0.0);
    if (j == 0) {
      W.blo[i] = dc(0.0);
      W.bup[i] = dc(0.0);
    }
  }
  __syncthreads();
  for (int l = L; l >= 0; --l) {  // wide layer l: 0 = prepend, else net layer l - 1
    const int t = l - 1;
    const int act = (l == 0) ? REACH_ACT_IDENTITY : N.acts[t];
    const int cols = (l == 0) ? nz + n : (t == 0 ? n : N.dims[t]);
    if (act != REACH_ACT_IDENTITY) {
      for (int j = tid; j < acols; j += kThreads) {
        D s, li, ui;
        bool boundary = false;
        if (!relax_d(act, W.pre[t][j], s, li, ui, boundary)) W.bad = 1;
        if (boundary) W.sub = 1;
        W.rel[0][j] = s;
        W.rel[1][j] = li;
        W.rel[2][j] = ui;
      }
      __syncthreads();
      if (W.bad) return 1;
    }
    // per output row i: the relaxation intercepts (ascending j) into b_lo / b_up, Lambda *= s, then
    // shift = matvec(Lambda_s, b) (linalg.hpp:40-51, 65-71) added to both.  The three chains of a row
    // are independent sequences, so they run on three different warps (lo: warp 0, up: warp 1, shift:
    // warp 2, which forms Lambda_s entries itself -- the same products), while the other warps write
    // Lambda_s into the spare buffer; each chain keeps the reference's order.
    const int src = (act != REACH_ACT_IDENTITY) ? (lb ^ 1) : lb;  // the buffer holding Lambda_s
    const int dst = src ^ 1;
    {
      const int wi = tid >> 5, ln = tid & 31;
      if (act != REACH_ACT_IDENTITY && wi < 2 && ln < n_o) {
        const int i = ln;
        D acc = (wi == 0) ? W.blo[i] : W.bup[i];
        for (int j = 0; j < acols; ++j) {
          const D aij = W.lam[lb][i][j];
          const bool pos = aij.v >= 0.0;
          // lower bound takes li for Lambda >= 0 (ui otherwise); upper bound the opposite
          const D r = W.rel[(pos == (wi == 0)) ? 1 : 2][j];
          acc = dadd(acc, dmul(aij, r));
        }
        if (wi == 0) W.blo[i] = acc;
        else W.bup[i] = acc;
      } else if (wi == 2 && ln < n_o) {
        const int i = ln;
        D acc = dc(0.0);
        for (int j = 0; j < acols; ++j) {
          const D bj = (l == 0) ? W.c[j] : (t == 0 ? W.bf0[j] : net.b(t, j));
          const D a = (act != REACH_ACT_IDENTITY) ? dmul(W.lam[lb][i][j], W.rel[0][j]) : W.lam[lb][i][j];
          acc = dadd(acc, dmul(a, bj));
        }
        W.shift[i] = acc;
      } else if (act != REACH_ACT_IDENTITY && wi >= 3) {
        for (int e = tid - 96; e < n_o * acols; e += kThreads - 96) {
          const int i = e / acols, j = e % acols;
          W.lam[src][i][j] = dmul(W.lam[lb][i][j], W.rel[0][j]);
        }
      }
    }
    __syncthreads();
    if (tid < n_o) {
      W.blo[tid] = dadd(W.blo[tid], W.shift[tid]);
      W.bup[tid] = dadd(W.bup[tid], W.shift[tid]);
    }
    // Lambda = matmul(Lambda_s, W_l) (linalg.hpp:53-63): element (i, j) sums k ascending, one thread per
    // element (consecutive threads = consecutive columns: coalesced W rows, Lambda entries broadcast).
    // (Measured: one thread per column with all rows' chains in registers is 13 % slower.)
    for (int e = tid; e < n_o * cols; e += kThreads) {
      const int i = e / cols, j = e % cols;
      D acc = dc(0.0);
      if (l == 0) {
        for (int k = 0; k < acols; ++k) {
          const D wkj = (j < nz) ? W.S[k][j] : dc(j - nz == k ? 1.0 : 0.0);
          acc = dadd(acc, dmul(W.lam[src][i][k], wkj));
        }
      } else if (net.sl != t) {  // no seeded parameter in this layer: plain constant weights
        const double* wcol = net.N.blob + net.N.w_off[t] + j;
        const int ld = net.N.ldw[t];
#pragma unroll 4
        for (int k = 0; k < acols; ++k) acc = dadd(acc, dmul(W.lam[src][i][k], dc(wcol[static_cast<long long>(k) * ld])));
      } else {
        for (int k = 0; k < acols; ++k) acc = dadd(acc, dmul(W.lam[src][i][k], net.w(t, k, j)));
      }
      W.lam[dst][i][j] = acc;
    }
    __syncthreads();
    lb = dst;
    acols = cols;
  }
  // tail (neural.hpp:383-391)
  for (int e = tid; e < n_o * nz; e += kThreads) W.oA[e / nz][e % nz] = W.lam[lb][e / nz][e % nz];
  for (int i = tid; i < n_o; i += kThreads) {
    const D mid = dmul(dadd(W.blo[i], W.bup[i]), dc(0.5));
    W.oc[i] = mid;
    DI rem{dsub(W.blo[i], mid), dsub(W.bup[i], mid)};
    for (int j = 0; j < n; ++j) rem = iadd(rem, iscale(W.lam[lb][i][nz + j], DI{dc(0.0), dc(0.0)}));
    W.orem[i] = rem;
  }
  __syncthreads();
  return 0;
}

// row_abs_sum (linalg.hpp:134-141) in Dual (reach::abs).
__device__ __forceinline__ D row_abs(const D* row, int cols) {
  D acc = dc(0.0);
  for (int j = 0; j < cols; ++j) acc = dadd(acc, dabs(row[j]));
  return acc;
}

// fold_overflow (flowpipe_ct.hpp:317-350) with a square G0 (dt_reach) by one warp: lane c < n + w holds
// column c of [G0 | Q1] in registers for the partial-pivot elimination (linalg.hpp:96-132; pivot column
// and factors broadcast from the lane owning column k); every element sees the reference's operation
// sequence.  The scalar tail (row abs-sums, G0.X - Q, column inflation, the queue shift) is lane-parallel
// over rows.  Called by all 32 lanes of warp 0 with identical nq.
__device__ __noinline__ void fold_warp_d(int n, int& nq, int cap, Work& W, int lane) {
  constexpr unsigned FULL = 0xffffffffu;
  while (nq > cap) {
    const int w = W.wid[0];
    const int ncol = n + w;
    int off_new = n;
    for (int q = 0; q + 1 < nq; ++q) off_new += W.wid[q];
    D col[kN];
#pragma unroll
    for (int i = 0; i < kN; ++i) col[i] = (lane < ncol && i < n) ? W.S[i][lane] : dc(0.0);
    if (lane < n) {
#pragma unroll
      for (int i = 0; i < kN; ++i)
        if (i < n) W.g0[i][lane] = col[i];
    } else if (lane < ncol) {
#pragma unroll
      for (int i = 0; i < kN; ++i)
        if (i < n) W.qa[i][lane - n] = col[i];
    }
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kN; ++k) {
      if (k >= n || !ok) break;
      int piv = k;
      double best = fabs(col[k].v);
#pragma unroll
      for (int i = k + 1; i < kN; ++i)
        if (i < n) {
          const double c = fabs(col[i].v);
          if (c > best) {
            best = c;
            piv = i;
          }
        }
      piv = __shfl_sync(FULL, piv, k);
      best = __shfl_sync(FULL, best, k);
      if (!(best > 1e-12)) {
        ok = false;
        break;
      }
#pragma unroll
      for (int r = k + 1; r < kN; ++r)
        if (r == piv) {
          const D t = col[k];
          col[k] = col[r];
          col[r] = t;
        }
      const bool upd = (lane >= k && lane < ncol);
#pragma unroll
      for (int i = k + 1; i < kN; ++i) {
        if (i < n) {
          D f = ddiv(col[i], col[k]);  // meaningful on lane k: a[i][k] / a[k][k]
          f.v = __shfl_sync(FULL, f.v, k);
          f.d = __shfl_sync(FULL, f.d, k);
          if (upd) col[i] = dsub(col[i], dmul(f, col[k]));
        }
      }
    }
    bool folded = false;
    if (ok) {
      // back substitution on the B lanes; a[i][k] comes from lane k
      D x[kN];
#pragma unroll
      for (int ii = kN - 1; ii >= 0; --ii) {
        if (ii < n) {
          D acc = col[ii];
#pragma unroll
          for (int k = ii + 1; k < kN; ++k)
            if (k < n) {
              D aik;
              aik.v = __shfl_sync(FULL, col[ii].v, k);
              aik.d = __shfl_sync(FULL, col[ii].d, k);
              acc = dsub(acc, dmul(aik, x[k]));
            }
          D aii;
          aii.v = __shfl_sync(FULL, col[ii].v, ii);
          aii.d = __shfl_sync(FULL, col[ii].d, ii);
          x[ii] = ddiv(acc, aii);
        } else {
          x[ii] = dc(0.0);
        }
      }
      if (lane >= n && lane < ncol) {
#pragma unroll
        for (int i = 0; i < kN; ++i)
          if (i < n) W.qx[i][lane - n] = x[i];
      }
      __syncwarp();
      if (lane < n) W.rr[lane] = dmul(row_abs(W.qx[lane], w), dc(1.0 + 1e-12));
      __syncwarp();
      double worst = 0.0;
      for (int j = 0; j < n; ++j) worst = (worst < W.rr[j].v) ? W.rr[j].v : worst;  // std::max on values
      if (worst <= 1.0) {
        for (int e = lane; e < n * w; e += 32) {
          const int i = e / w, j = e % w;
          D acc = dc(0.0);
          for (int k = 0; k < n; ++k) acc = dadd(acc, dmul(W.g0[i][k], W.qx[k][j]));
          W.qe[i][j] = dsub(acc, W.qa[i][j]);
        }
        __syncwarp();
        for (int e = lane; e < n * n; e += 32) {
          const int i = e / n, j = e % n;
          W.S[i][j] = dmul(W.S[i][j], dadd(dc(1.0), W.rr[j]));
        }
        if (lane < n)
          W.S[lane][off_new + lane] =
              dadd(W.S[lane][off_new + lane], dmul(row_abs(W.qe[lane], w), dc(1.0 + 1e-12)));
        folded = true;
      }
    }
    if (!folded && lane < n) W.S[lane][off_new + lane] = dadd(W.S[lane][off_new + lane], row_abs(&W.S[lane][n], w));
    __syncwarp();
    int total = n;
    for (int q = 0; q < nq; ++q) total += W.wid[q];
    if (lane < n)
      for (int j = n; j + w < total; ++j) W.S[lane][j] = W.S[lane][j + w];
    __syncwarp();
    if (lane == 0)
      for (int q = 0; q + 1 < nq; ++q) W.wid[q] = W.wid[q + 1];
    __syncwarp();
    --nq;
  }
}

// Constraint::margin (mpc.hpp:40-86) in Dual on tube box t.
__device__ inline D margin_d(const PlanParams& P, const DevConstraint& c, const D* lo, const D* hi) {
  const int* dims = P.ibuf + c.dims_off;
  const double* dv = P.dbuf;
  switch (c.type) {
    case 0: {
      D worst = dc(c.b);
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        const double aj = dv[c.a_off + j];
        const D term = aj >= 0.0 ? dmul(hi[d], dc(aj)) : dmul(lo[d], dc(aj));
        worst = dsub(worst, term);
      }
      return worst;
    }
    case 1: {
      D d2 = dc(0.0);
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        const double cj = dv[c.c_off + j];
        D gap = dc(0.0);
        if (lo[d].v > cj) gap = dsub(lo[d], dc(cj));
        else if (hi[d].v < cj) gap = dsub(dc(cj), hi[d]);
        d2 = dadd(d2, dmul(gap, gap));
      }
      return dsub(dsqrt(d2), dc(c.radius));
    }
    case 2: {
      D worst = dc(__longlong_as_double(0x7ff0000000000000ll));
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        worst = dmin(worst, dsub(lo[d], dc(dv[c.lo_off + j])));
        worst = dmin(worst, dsub(dc(dv[c.hi_off + j]), hi[d]));
      }
      return worst;
    }
    default: {
      D v = dc(0.0);
      for (int j = 0; j < c.k; ++j) v = dadd(v, dsub(hi[dims[j]], lo[dims[j]]));
      return dsub(dc(c.vmax), v);
    }
  }
}

// dt_reach (dt_reach.hpp:41-104) in Dual from the box W.tlo[0] / W.thi[0]
// (written and synchronized by the caller) under the actions W.acts, by the
// whole CTA.  Returns the number of boxes pushed; `failed` = the tube was
// marked failed (a relax_activation throw, a diverged certification or a
// diverged box).
__device__ __forceinline__ int dt_tube_d(const NetView& net, int n, int m, int H, int window, int rebuild, Work& W, int tid,
                                bool& failed) {
  const DevNet& N = net.N;
  failed = false;
  const int cap = window > 0 ? window : 1;
  auto init_state = [&](const D* lo, const D* hi) {
    for (int e = tid; e < n * n; e += kThreads) {
      const int i = e / n, q = e % n;
      if (q == 0) W.c[i] = dmul(dadd(lo[i], hi[i]), dc(0.5));
      W.S[i][q] = (i == q) ? dmul(dsub(hi[i], lo[i]), dc(0.5)) : dc(0.0);
    }
  };
  if (tid == 0) {
    W.nq = 0;
    W.stop = 0;
  }
  __syncthreads();
  init_state(W.tlo[0], W.thi[0]);
  int nb = 1;
  for (int k = 0; k < H; ++k) {
    // freeze_trailing_inputs (neural.hpp:398-413)
    for (int u = tid; u < N.dims[1]; u += kThreads) {
      D bb = net.b(0, u);
      for (int q = 0; q < m; ++q) bb = dadd(bb, dmul(net.w(0, u, n + q), W.acts[k][q]));
      W.bf0[u] = bb;
    }
    __syncthreads();
    const int nq = W.nq;
    int nz = n;
    for (int q = 0; q < nq; ++q) nz += W.wid[q];
    if (certify_d(net, n, nz, W, tid)) {  // relax_activation throws: tube failed at k
      failed = true;
      break;
    }
    if (tid == 0) {
      bool rfin = true;
      for (int i = 0; i < n; ++i) rfin = rfin && dfin(W.orem[i].lo) && dfin(W.orem[i].hi);
      W.stop = rfin ? 0 : 1;
    }
    __syncthreads();
    if (W.stop) {  // diverged certification
      failed = true;
      break;
    }
    // re-seed (dt_reach.hpp:69-92)
    for (int e = tid; e < n * (nz + n); e += kThreads) {
      const int i = e / (nz + n), q = e % (nz + n);
      if (q == 0) W.c[i] = dadd(W.oc[i], imid(W.orem[i]));
      W.S[i][q] = q < nz ? W.oA[i][q] : (q - nz == i ? irad(W.orem[i]) : dc(0.0));
    }
    __syncthreads();
    if (tid < 32) {  // fold_overflow by warp 0
      if (tid == 0) W.wid[nq] = n;
      __syncwarp();
      int nq2 = nq + 1;
      fold_warp_d(n, nq2, cap, W, tid);
      if (tid == 0) W.nq = nq2;
    }
    __syncthreads();
    // symbolic_box (flowpipe_ct.hpp:413-424)
    for (int i = tid; i < n; i += kThreads) {
      D r = row_abs(W.S[i], n);
      int off = n;
      for (int q = 0; q < W.nq; ++q) {
        r = dadd(r, row_abs(&W.S[i][off], W.wid[q]));
        off += W.wid[q];
      }
      W.tlo[k + 1][i] = dsub(W.c[i], r);
      W.thi[k + 1][i] = dadd(W.c[i], r);
    }
    __syncthreads();
    if (tid == 0) {
      bool fin = true;
      for (int i = 0; i < n; ++i) fin = fin && dfin(W.tlo[k + 1][i]) && dfin(W.thi[k + 1][i]);
      W.stop = fin ? 0 : 1;
      if (fin && rebuild) W.nq = 0;
    }
    __syncthreads();
    nb = k + 2;
    if (W.stop) {  // diverged box (pushed)
      failed = true;
      break;
    }
    if (rebuild) {
      init_state(W.tlo[k + 1], W.thi[k + 1]);
      __syncthreads();
    }
  }
  return nb;
}

// plan_objective (mpc.hpp:158-208) in Dual, seeded on action component
// j = blockIdx.x; one CTA per direction, the working set in shared memory.
__global__ void __launch_bounds__(kThreads, 2) plan_grad_kernel(const GradArgs G) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Work& W = *reinterpret_cast<Work*>(smem_raw);
  const int j = blockIdx.x, tid = threadIdx.x;
  const PlanParams& P = G.P;
  const int H = P.H, n = P.n, m = P.m;
  const NetView net{P.net};
  const DevNet& N = P.net;
  const int L = N.L;
  for (int e = tid; e < H * m; e += kThreads) W.acts[e / m][e % m] = D{G.base[e], e == j ? 1.0 : 0.0};
  if (tid == 0) {
    W.obj = dc(0.0);
    W.sub = 0;
  }
  for (int i = tid; i < n; i += kThreads) W.hb[0][i].lo = dc(P.x0[i]);
  __syncthreads();
  // nominal rollout + stage costs (mpc.hpp:170-184), MLPNet::forward (neural.hpp:58-76)
  int cur = 0;
  for (int t = 0; t < H; ++t) {
    for (int i = tid; i < m; i += kThreads) W.hb[cur][n + i].lo = W.acts[t][i];
    __syncthreads();
    for (int l = 0; l < L; ++l) {
      const int rows = N.dims[l + 1], cols = N.dims[l];
      for (int u = tid; u < rows; u += kThreads) {
        D acc = dc(0.0);
        if (l + 1 < L)
          for (int q = 0; q < cols; ++q) acc = dadd(acc, dmul(net.wt(l, u, q), W.hb[cur][q].lo));
        else
          for (int q = 0; q < cols; ++q) acc = dadd(acc, dmul(net.w(l, u, q), W.hb[cur][q].lo));
        D h = dadd(acc, net.b(l, u));
        if (N.acts[l] == REACH_ACT_RELU) {
          if (h.v < 0.0) h = dc(0.0);
        } else if (N.acts[l] == REACH_ACT_TANH) {
          h = dtanh(h);
        }
        W.hb[cur ^ 1][u].lo = h;
      }
      cur ^= 1;
      __syncthreads();
    }
    if (tid == 0) {
      D obj = W.obj;
      for (int i = 0; i < m; ++i) obj = dadd(obj, dmul(dmul(dc(P.r_w[i]), W.acts[t][i]), W.acts[t][i]));
      for (int i = 0; i < n; ++i) {
        const D dd = dsub(W.hb[cur][i].lo, dc(P.x_goal[i]));
        obj = dadd(obj, dmul(dmul(dc(P.q_w[i]), dd), dd));
      }
      W.obj = obj;
    }
    // x_{t+1} stays in hb[cur][0..n); the next step appends its action behind it
  }
  __syncthreads();
  // dt_reach (dt_reach.hpp:41-104) at radius eps around x0 (box_from_center, interval.hpp:224-235)
  if (tid == 0)
    for (int i = 0; i < n; ++i) {
      const D c0 = dc(P.x0[i]), r0 = dc(G.eps);
      W.tlo[0][i] = dsub(c0, r0);
      W.thi[0][i] = dadd(c0, r0);
    }
  __syncthreads();
  bool failed = false;
  const int nb = dt_tube_d(net, n, m, H, G.window, G.rebuild, W, tid, failed);
  // constraint penalties over the tube (mpc.hpp:187-200)
  if (tid == 0) {
    D obj = W.obj;
    for (int t = 1; t <= H; ++t) {
      bool ok = t < nb;
      for (int i = 0; ok && i < n; ++i) ok = dfin(W.tlo[t][i]) && dfin(W.thi[t][i]);
      if (ok) {
        for (int q = 0; q < P.n_con; ++q) {
          const D g = margin_d(P, P.con[q], W.tlo[t], W.thi[t]);
          obj = dadd(obj, dmul(dc(P.penalty), dmax(dc(0.0), dneg(g))));
        }
      } else if (P.n_con > 0) {
        obj = dadd(obj, dc(P.penalty * P.diverged_margin * static_cast<double>(P.n_con)));
      }
    }
    G.grad[j] = obj.d;
    G.value[j] = obj.v;
  }
}

// ---------------------------------------------------------------------------
// grad_tube_volume (refine.hpp:263-311): d tube_volume(dt_reach(...)) / d p for
// p = the X0 centre (radii fixed), the flat action sequence, or the network
// parameters in net_params order (neural.hpp:133-140).  One CTA per pass:
//   forward_dual (grad_forward, refine.hpp:186-207): CTA j seeds p_j;
//   finite_difference (grad_fd, refine.hpp:209-231): CTAs 2j / 2j+1 evaluate
//   p_j +/- h, h = rel_step * max(1, |p_j|); the last CTA is the unperturbed pass
//   (f0 and the branch-boundary flag, as in the reference).
enum : int { TARGET_X0_CENTER = 0, TARGET_ACTIONS = 1, TARGET_WEIGHTS = 2 };

struct VolArgs {
  DevNet net;
  int n, m, H, window, rebuild;
  const double* center;   // [n]  box_center(x0)
  const double* radius;   // [n]  box_radius(x0)
  const double* actions;  // [H*m]
  int target, dim, fd;  // dim = the passes' parameter count (a slice [p0, p0 + dim) of the target)
  long long p0;
  double rel_step;
  long long poff[kMaxLayers + 1];  // net_params offset of each layer's W (then its b)
  double* value;          // [passes] tube volume (primal) seen by each pass
  double* tangent;        // [passes]
  int* sub;               // [1] any pass noted a branch boundary (forward) / the f0 pass did (fd)
};

__global__ void __launch_bounds__(kThreads, 2) tube_volume_grad_kernel(const VolArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Work& W = *reinterpret_cast<Work*>(smem_raw);
  const int tid = threadIdx.x, pass = blockIdx.x;
  const int n = A.n, m = A.m, H = A.H;
  // which parameter this pass moves, by how much, with which tangent
  int p = -1;
  double delta = 0.0, seed = 0.0;
  if (!A.fd) {
    p = static_cast<int>(A.p0 + pass);
    seed = 1.0;
  } else if (pass < 2 * A.dim) {
    p = static_cast<int>(A.p0 + (pass >> 1));
  }
  NetView net{A.net};
  double x = 0.0;
  if (p >= 0) {
    if (A.target == TARGET_X0_CENTER) {
      x = A.center[p];
    } else if (A.target == TARGET_ACTIONS) {
      x = A.actions[p];
    } else {
      int l = 0;
      while (l + 1 <= A.net.L && A.poff[l + 1] <= p) ++l;
      const long long q = p - A.poff[l];
      const int rows = A.net.dims[l + 1], cols = A.net.dims[l];
      net.sl = l;
      if (q < static_cast<long long>(rows) * cols) {
        net.si = static_cast<int>(q / cols);
        net.sj = static_cast<int>(q % cols);
        x = A.net.blob[A.net.w_off[l] + static_cast<long long>(net.si) * A.net.ldw[l] + net.sj];
      } else {
        net.si = static_cast<int>(q - static_cast<long long>(rows) * cols);
        net.sj = -1;
        x = A.net.blob[A.net.b_off[l] + net.si];
      }
    }
    if (A.fd) {
      const double h = mul(A.rel_step, fmax(1.0, fabs(x)));
      delta = (pass & 1) ? -h : h;
    }
    net.delta = delta;
    net.seed = seed;
  }
  auto param = [&](double v, int target, int idx) -> D {
    if (A.target != target || idx != p) return dc(v);
    return D{delta != 0.0 ? add(v, delta) : v, seed};
  };
  for (int e = tid; e < H * m; e += kThreads) W.acts[e / m][e % m] = param(A.actions[e], TARGET_ACTIONS, e);
  if (tid == 0) {
    W.sub = 0;
    for (int i = 0; i < n; ++i) {  // box_from_center(c, radius) (interval.hpp:224-235)
      const D c = param(A.center[i], TARGET_X0_CENTER, i), r = dc(A.radius[i]);
      W.tlo[0][i] = dsub(c, r);
      W.thi[0][i] = dadd(c, r);
    }
  }
  __syncthreads();
  bool failed = false;
  const int nb = dt_tube_d(net, n, m, H, A.window, A.rebuild, W, tid, failed);
  if (tid == 0) {
    // tube_volume (tube.hpp:40-46): +inf once diverged; else the sum of box width sums
    D acc = dc(0.0);
    bool fin = !failed;
    for (int k = 0; fin && k < nb; ++k) {
      D v = dc(0.0);
      for (int i = 0; i < n; ++i) {
        fin = fin && dfin(W.tlo[k][i]) && dfin(W.thi[k][i]);
        v = dadd(v, dsub(W.thi[k][i], W.tlo[k][i]));
      }
      acc = dadd(acc, v);
    }
    if (!fin) acc = dc(__longlong_as_double(0x7ff0000000000000ll));
    A.value[pass] = acc.v;
    A.tangent[pass] = acc.d;
    const bool counts = !A.fd || pass == 2 * A.dim;
    if (counts && W.sub) atomicOr(A.sub, 1);
  }
}

// ---------------------------------------------------------------------------
// reach_loss (training.hpp:99-126): (1/M) sum_m [diverged ? cap : log(1 + predicted_volume(tube_m))],
// tube_m = dt_reach from box_from_center(x0_m, eps) under the episode's first t_h actions.  CTA
// (pass, episode): pass p seeds network parameter p (net_params order) for grad_forward over the
// parameters (the training objective's gradient); pass -1 (value only) seeds nothing.  The per-episode
// Dual terms are combined on the host in episode order, as the reference's accumulator does.
struct LossArgs {
  DevNet net;
  int n, m, H, window, rebuild, M;
  const double* x0;       // [M][n] episode start states
  const double* actions;  // [M][H][m]
  double eps, cap;
  int seeded;             // 0: value only (one pass, no seed)
  long long poff[kMaxLayers + 1];
  double* term_v;         // [passes][M]
  double* term_d;
  int* diverged;          // [M] (pass 0)
};

__global__ void __launch_bounds__(kThreads, 2) reach_loss_grad_kernel(const LossArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Work& W = *reinterpret_cast<Work*>(smem_raw);
  const int tid = threadIdx.x, pass = blockIdx.x, ep = blockIdx.y;
  const int n = A.n, m = A.m, H = A.H;
  NetView net{A.net};
  if (A.seeded) {
    const long long p = pass;
    int l = 0;
    while (l + 1 <= A.net.L && A.poff[l + 1] <= p) ++l;
    const long long q = p - A.poff[l];
    const int rows = A.net.dims[l + 1], cols = A.net.dims[l];
    net.sl = l;
    if (q < static_cast<long long>(rows) * cols) {
      net.si = static_cast<int>(q / cols);
      net.sj = static_cast<int>(q % cols);
    } else {
      net.si = static_cast<int>(q - static_cast<long long>(rows) * cols);
      net.sj = -1;
    }
    net.seed = 1.0;
  }
  const double* acts = A.actions + static_cast<size_t>(ep) * H * m;
  for (int e = tid; e < H * m; e += kThreads) W.acts[e / m][e % m] = dc(acts[e]);
  if (tid == 0) {
    W.sub = 0;
    for (int i = 0; i < n; ++i) {  // box_from_center(x0, S(eps))
      const D c = dc(A.x0[static_cast<size_t>(ep) * n + i]), r = dc(A.eps);
      W.tlo[0][i] = dsub(c, r);
      W.thi[0][i] = dadd(c, r);
    }
  }
  __syncthreads();
  bool failed = false;
  const int nb = dt_tube_d(net, n, m, H, A.window, A.rebuild, W, tid, failed);
  if (tid == 0) {
    bool div = failed;
    for (int k = 0; !div && k < nb; ++k)
      for (int i = 0; i < n; ++i) div = div || !(dfin(W.tlo[k][i]) && dfin(W.thi[k][i]));
    D term;
    if (div) {
      term = dc(A.cap);
    } else {
      D v = dc(0.0);  // predicted_volume (training.hpp:89-93): boxes 1..
      for (int k = 1; k < nb; ++k) {
        D b = dc(0.0);
        for (int i = 0; i < n; ++i) b = dadd(b, dsub(W.thi[k][i], W.tlo[k][i]));
        v = dadd(v, b);
      }
      const D a = dadd(dc(1.0), v);
      term = D{log(a.v), __ddiv_rn(a.d, a.v)};  // reach::log (scalar.hpp:47)
    }
    const size_t o = static_cast<size_t>(pass) * A.M + ep;
    A.term_v[o] = term.v;
    A.term_d[o] = term.d;
    if (pass == 0) A.diverged[ep] = div ? 1 : 0;
  }
}

// Seeds network parameter p (net_params order, neural.hpp:133-140) in a NetView.
__device__ __forceinline__ void seed_param(NetView& net, const long long* poff, long long p) {
  int l = 0;
  while (l + 1 <= net.N.L && poff[l + 1] <= p) ++l;
  const long long q = p - poff[l];
  const int rows = net.N.dims[l + 1], cols = net.N.dims[l];
  net.sl = l;
  if (q < static_cast<long long>(rows) * cols) {
    net.si = static_cast<int>(q / cols);
    net.sj = static_cast<int>(q % cols);
  } else {
    net.si = static_cast<int>(q - static_cast<long long>(rows) * cols);
    net.sj = -1;
  }
  net.seed = 1.0;
}

// ---------------------------------------------------------------------------
// pred_loss (training.hpp:60-83): the autoregressive multi-step prediction loss and its grad_forward
// over the model's parameters.  One CTA per (pass p, episode e): the nominal rollout
// xhat_{t+1} = model.forward([xhat_t; u_t]) in reach::Dual with parameter p seeded (pass 0 of a
// value-only launch: nothing seeded), emitting each step's term w_t * ||xhat_{t+1} - x_{t+1}||^2
// (Dual); the host sums the terms in the reference's (episode, step) order.
constexpr int kPredW = 256;  // widest layer
constexpr int kPredThreads = 128;

struct PredArgs {
  DevNet net;
  int n, m, T, M, seeded;
  long long poff[kMaxLayers + 1];
  const double* states;   // [M][Ls + 1][n]
  const double* actions;  // [M][Ls][m]
  int ls;                 // stored episode length Ls >= T
  const double* weights;  // [T]
  double* term_v;         // [passes][M][T]
  double* term_d;
};

__global__ void __launch_bounds__(kPredThreads) pred_loss_grad_kernel(const PredArgs A) {
  __shared__ D hb[2][kPredW];
  const int tid = threadIdx.x, pass = blockIdx.x, ep = blockIdx.y;
  const int n = A.n, m = A.m, T = A.T;
  NetView net{A.net};
  if (A.seeded) seed_param(net, A.poff, pass);
  const DevNet& N = A.net;
  const double* st = A.states + static_cast<size_t>(ep) * (A.ls + 1) * n;
  const double* ac = A.actions + static_cast<size_t>(ep) * A.ls * m;
  for (int i = tid; i < n; i += kPredThreads) hb[0][i] = dc(st[i]);
  int cur = 0;
  for (int t = 0; t < T; ++t) {
    for (int i = tid; i < m; i += kPredThreads) hb[cur][n + i] = dc(ac[static_cast<size_t>(t) * m + i]);
    __syncthreads();
    for (int l = 0; l < N.L; ++l) {  // MLPNet::forward (neural.hpp:58-76), matvec (linalg.hpp:41-51)
      const int rows = N.dims[l + 1], cols = N.dims[l];
      for (int u = tid; u < rows; u += kPredThreads) {
        D acc = dc(0.0);
        if (l + 1 < N.L)
          for (int q = 0; q < cols; ++q) acc = dadd(acc, dmul(net.wt(l, u, q), hb[cur][q]));
        else
          for (int q = 0; q < cols; ++q) acc = dadd(acc, dmul(net.w(l, u, q), hb[cur][q]));
        D h = dadd(acc, net.b(l, u));
        if (N.acts[l] == REACH_ACT_RELU) {
          if (h.v < 0.0) h = dc(0.0);
        } else if (N.acts[l] == REACH_ACT_TANH) {
          h = dtanh(h);
        }
        hb[cur ^ 1][u] = h;
      }
      cur ^= 1;
      __syncthreads();
    }
    if (tid == 0) {
      const double* tgt = st + static_cast<size_t>(t + 1) * n;
      D err = dc(0.0);
      for (int j = 0; j < n; ++j) {
        const D d = dsub(hb[cur][j], dc(tgt[j]));
        err = dadd(err, dmul(d, d));
      }
      const D term = dmul(dc(A.weights[t]), err);
      const size_t o = (static_cast<size_t>(pass) * A.M + ep) * T + t;
      A.term_v[o] = term.v;
      A.term_d[o] = term.d;
    }
    // xhat_{t+1} stays in hb[cur][0..n); the next step appends its action behind it
  }
}

// ---------------------------------------------------------------------------
// track_loss (training.hpp:134-178) with the quadrotor plant (systems.hpp:22-64) and its grad_forward
// over the controller's parameters.  One CTA per (pass p, episode e): uhat = controller([xhat; y_ref_t])
// (zero-order hold), rk4_substeps fixed RK4 steps (ode.hpp:76-91) of the plant under uhat, the
// weighted errors; the episode's Dual sum (or the cap if it blew up) goes to the host, which sums the
// episodes in order.  sin / cos / tanh are CUDA's (the reference uses glibc's): values within ulps.
__device__ __forceinline__ D dsin(D a) { return D{sin(a.v), mul(cos(a.v), a.d)}; }
__device__ __forceinline__ D dcos(D a) { return D{cos(a.v), mul(-sin(a.v), a.d)}; }

struct TrackArgs {
  DevNet net;             // controller
  int n, l, r, T, M, seeded, rk4;
  long long poff[kMaxLayers + 1];
  double prm[5];          // QuadrotorParams {mass, gravity, jx, jy, jz}
  double gamma, delta, cap;
  const double* states;   // [M][Ls + 1][n]
  const double* actions;  // [M][Ls][l] logged controls
  const double* y_ref;    // [M][Ls][r] or null
  int ls;
  const double* weights;  // [T]
  double* ep_v;           // [passes][M] episode term (Dual)
  double* ep_d;
  int* blown;             // [M] (pass 0)
};

// quadrotor_ode (systems.hpp:24-64) in Dual, operation for operation
__device__ inline void quad_ode_d(const D* x, const D* u, const double* prm, D* dx) {
  const D vx = x[3], vy = x[4], vz = x[5], phi = x[6], theta = x[7], psi = x[8], p = x[9], q = x[10], r = x[11];
  const D sphi = dsin(phi), cphi = dcos(phi), sth = dsin(theta), cth = dcos(theta), spsi = dsin(psi),
          cpsi = dcos(psi);
  const D b3x = dadd(dmul(dmul(cphi, sth), cpsi), dmul(sphi, spsi));
  const D b3y = dsub(dmul(dmul(cphi, sth), spsi), dmul(sphi, cpsi));
  const D b3z = dmul(cphi, cth);
  const double mass = prm[0], g = prm[1], jx = prm[2], jy = prm[3], jz = prm[4];
  const D a = dmul(u[0], dc(1.0 / mass));
  dx[0] = vx;
  dx[1] = vy;
  dx[2] = vz;
  dx[3] = dmul(a, b3x);
  dx[4] = dmul(a, b3y);
  dx[5] = dsub(dmul(a, b3z), dc(g));
  const D tth = ddiv(sth, cth);
  dx[6] = dadd(dadd(p, dmul(dmul(sphi, tth), q)), dmul(dmul(cphi, tth), r));
  dx[7] = dsub(dmul(cphi, q), dmul(sphi, r));
  dx[8] = dadd(dmul(ddiv(sphi, cth), q), dmul(ddiv(cphi, cth), r));
  dx[9] = dadd(dmul(dmul(q, r), dc((jy - jz) / jx)), dmul(u[1], dc(1.0 / jx)));
  dx[10] = dadd(dmul(dmul(p, r), dc((jz - jx) / jy)), dmul(u[2], dc(1.0 / jy)));
  dx[11] = dadd(dmul(dmul(p, q), dc((jx - jy) / jz)), dmul(u[3], dc(1.0 / jz)));
}

__global__ void __launch_bounds__(kPredThreads) track_loss_grad_kernel(const TrackArgs A) {
  __shared__ D hb[2][kPredW];
  __shared__ D xs[16], us[8];
  __shared__ int s_blown;
  const int tid = threadIdx.x, pass = blockIdx.x, ep = blockIdx.y;
  const int n = A.n, l = A.l, r = A.r, T = A.T;
  NetView net{A.net};
  if (A.seeded) seed_param(net, A.poff, pass);
  const DevNet& N = A.net;
  const double* st = A.states + static_cast<size_t>(ep) * (A.ls + 1) * n;
  const double* ul = A.actions + static_cast<size_t>(ep) * A.ls * l;
  const double* yr = A.y_ref ? A.y_ref + static_cast<size_t>(ep) * A.ls * r : nullptr;
  if (tid < n) xs[tid] = dc(st[tid]);
  D ep_acc = dc(0.0);
  if (tid == 0) s_blown = 0;
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    if (s_blown) break;
    // in = xhat (+ y_ref_t); uhat = controller.forward(in) (neural.hpp:58-76)
    for (int i = tid; i < n; i += kPredThreads) hb[0][i] = xs[i];
    if (yr)
      for (int i = tid; i < r; i += kPredThreads) hb[0][n + i] = dc(yr[static_cast<size_t>(t) * r + i]);
    __syncthreads();
    int cur = 0;
    for (int q = 0; q < N.L; ++q) {
      const int rows = N.dims[q + 1], cols = N.dims[q];
      for (int u = tid; u < rows; u += kPredThreads) {
        D acc = dc(0.0);
        if (q + 1 < N.L)
          for (int k = 0; k < cols; ++k) acc = dadd(acc, dmul(net.wt(q, u, k), hb[cur][k]));
        else
          for (int k = 0; k < cols; ++k) acc = dadd(acc, dmul(net.w(q, u, k), hb[cur][k]));
        D h = dadd(acc, net.b(q, u));
        if (N.acts[q] == REACH_ACT_RELU) {
          if (h.v < 0.0) h = dc(0.0);
        } else if (N.acts[q] == REACH_ACT_TANH) {
          h = dtanh(h);
        }
        hb[cur ^ 1][u] = h;
      }
      cur ^= 1;
      __syncthreads();
    }
    if (tid == 0) {
      D err_u = dc(0.0);
      for (int j = 0; j < l; ++j) {
        us[j] = hb[cur][j];
        const D d = dsub(us[j], dc(ul[static_cast<size_t>(t) * l + j]));
        err_u = dadd(err_u, dmul(d, d));
      }
      // rk4_substeps RK4 steps of h = delta / substeps (ode.hpp:76-91)
      const double h = A.delta / A.rk4;
      D x[12], k1[12], k2[12], k3[12], k4[12], tmp[12];
      for (int i = 0; i < 12; ++i) x[i] = xs[i];
      for (int ss = 0; ss < A.rk4; ++ss) {
        quad_ode_d(x, us, A.prm, k1);
        for (int i = 0; i < 12; ++i) tmp[i] = dadd(x[i], dmul(dc(h * 0.5), k1[i]));
        quad_ode_d(tmp, us, A.prm, k2);
        for (int i = 0; i < 12; ++i) tmp[i] = dadd(x[i], dmul(dc(h * 0.5), k2[i]));
        quad_ode_d(tmp, us, A.prm, k3);
        for (int i = 0; i < 12; ++i) tmp[i] = dadd(x[i], dmul(dc(h), k3[i]));
        quad_ode_d(tmp, us, A.prm, k4);
        for (int i = 0; i < 12; ++i)
          x[i] = dadd(x[i], dmul(dc(h / 6.0), dadd(dadd(dadd(k1[i], dmul(dc(2.0), k2[i])), dmul(dc(2.0), k3[i])), k4[i])));
      }
      D err_x = dc(0.0);
      const double* xl = st + static_cast<size_t>(t + 1) * n;
      for (int j = 0; j < n; ++j) {
        xs[j] = x[j];
        const D d = dsub(x[j], dc(xl[j]));
        err_x = dadd(err_x, dmul(d, d));
      }
      ep_acc = dadd(ep_acc, dmul(dc(A.weights[t]), dadd(err_u, dmul(dc(A.gamma), err_x))));
      if (!isfinite(ep_acc.v)) s_blown = 1;
    }
    __syncthreads();
  }
  if (tid == 0) {
    const D term = s_blown ? dc(A.cap) : ep_acc;
    const size_t o = static_cast<size_t>(pass) * A.M + ep;
    A.ep_v[o] = term.v;
    A.ep_d[o] = term.d;
    if (pass == 0) A.blown[ep] = s_blown;
  }
}

}  // namespace dual
}  // namespace rb
