// Reachability-aware MPC objective on the device (mpc.hpp:40-202).
//
// plan_eval = nominal rollout through the one-step network + quadratic stage
// costs, then constraint penalties over the certified tube (computed by the
// DT horizon kernel), all in the reference's operation order with separate
// multiply / add roundings.
#pragma once

#include "dt_common.cuh"
#include "dt_kernel.cuh"

namespace rb {

constexpr int kMaxConstraints = 16;

struct DevConstraint {
  int type, k;       // k = number of dims the constraint reads
  int dims_off;      // offsets into PlanParams::ibuf / dbuf
  int a_off, c_off, lo_off, hi_off;
  double b, radius, vmax;
};

struct PlanParams {
  DevNet net;
  int B, H, n, m;
  const double* x0;       // [n]
  const double* actions;  // [B][H][m]
  const double* x_goal;   // [n]   (in dbuf)
  const double* q_w;
  const double* r_w;
  int n_con;
  DevConstraint con[kMaxConstraints];
  const int* ibuf;
  const double* dbuf;
  double penalty, diverged_margin;
  // tube produced by the DT kernel
  const double* tube_lo;  // [B][H+1][n]
  const double* tube_hi;
  const int* n_boxes;
  const int* status;
  double* objective;      // [B]
  int* diverged;          // [B]
};

// Constraint::margin (mpc.hpp:40-86) on box k of candidate b.
__device__ inline double con_margin(const PlanParams& P, const DevConstraint& c, const double* lo, const double* hi) {
  const int* dims = P.ibuf + c.dims_off;
  const double* dv = P.dbuf;
  switch (c.type) {
    case 0: {  // halfspace_avoid: b - max_{y in box} a.y
      double worst = c.b;
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        const double aj = dv[c.a_off + j];
        const double term = aj >= 0.0 ? mul(hi[d], aj) : mul(lo[d], aj);
        worst = sub(worst, term);
      }
      return worst;
    }
    case 1: {  // sphere_avoid: box-to-center distance minus radius
      double d2 = 0.0;
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        const double cj = dv[c.c_off + j];
        double gap = 0.0;
        if (lo[d] > cj) gap = sub(lo[d], cj);
        else if (hi[d] < cj) gap = sub(cj, hi[d]);
        d2 = add(d2, mul(gap, gap));
      }
      return sub(__dsqrt_rn(d2), c.radius);
    }
    case 2: {  // box_stay_in: worst slack
      double worst = __longlong_as_double(0x7ff0000000000000ll);
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        worst = smin(worst, sub(lo[d], dv[c.lo_off + j]));
        worst = smin(worst, sub(dv[c.hi_off + j], hi[d]));
      }
      return worst;
    }
    default: {  // max_volume
      double v = 0.0;
      for (int j = 0; j < c.k; ++j) {
        const int d = dims[j];
        v = add(v, sub(hi[d], lo[d]));
      }
      return sub(c.vmax, v);
    }
  }
}

// One warp per candidate, kPlanWarps candidates per block.  Per step and
// layer the block stages W_l^T once in shared memory (coalesced), then every
// warp runs the layer with lanes over output units, each output a sequential
// dot product over the inputs exactly as MLPNet::forward's matvec
// (linalg.hpp:40-51); lane 0 sums the objective in the reference's order.
constexpr int kPlanWarps = 16;

__global__ void __launch_bounds__(kPlanWarps * 32) plan_objective_kernel(const PlanParams P, int vec, int wmax) {
  extern __shared__ __align__(16) double psm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b = blockIdx.x * kPlanWarps + warp;
  const bool live = b < P.B;
  double* wsm = psm;                                      // staged W_l^T: cols x rows (ld = rows)
  double* vin = psm + wmax + static_cast<size_t>(warp) * 2 * vec;
  double* vout = vin + vec;
  const DevNet& N = P.net;
  const int n = P.n, m = P.m, H = P.H, L = N.L;
  const double* acts = P.actions + static_cast<size_t>(live ? b : 0) * H * m;
  double x_reg = (lane < n) ? P.x0[lane] : 0.0;  // lane d holds x_d between steps
  double obj = 0.0;                               // lane 0's running objective
  for (int t = 0; t < H; ++t) {
    const double* u = acts + static_cast<size_t>(t) * m;
    if (lane < n) vin[lane] = x_reg;
    for (int j = lane; j < m; j += 32) vin[n + j] = u[j];
    double* a = vin;
    double* o = vout;
    for (int l = 0; l < L; ++l) {
      const int rows = N.dims[l + 1], cols = N.dims[l];
      const double* wt = N.blob + N.wt_off[l];
      const int ld = N.ldt[l];
      __syncthreads();  // previous layer done with wsm
      for (int q = threadIdx.x; q < cols * rows; q += blockDim.x) {
        const int j = q / rows, oo = q % rows;
        wsm[q] = __ldg(wt + static_cast<size_t>(j) * ld + oo);
      }
      __syncthreads();
      const double* bias = N.blob + N.b_off[l];
      const int act = N.acts[l];
      for (int o0 = lane; o0 < rows; o0 += 32) {
        double acc = 0.0;
        for (int j = 0; j < cols; ++j) acc = add(acc, mul(wsm[j * rows + o0], a[j]));
        double v = add(acc, __ldg(bias + o0));
        if (act == 0) v = (v < 0.0) ? 0.0 : v;  // MLPNet::h_relu (neural.hpp:85-87)
        else if (act == 1) v = tanh(v);
        o[o0] = v;
      }
      __syncwarp();
      double* tmp = a;
      a = o;
      o = tmp;
    }
    if (lane < n) x_reg = a[lane];
    if (lane == 0) {  // stage costs (mpc.hpp:171-183)
      for (int j = 0; j < m; ++j) obj = add(obj, mul(mul(P.r_w[j], u[j]), u[j]));
      for (int j = 0; j < n; ++j) {
        const double d = sub(a[j], P.x_goal[j]);
        obj = add(obj, mul(mul(P.q_w[j], d), d));
      }
    }
    __syncwarp();
  }
  if (lane != 0 || !live) return;
  const int nb = P.n_boxes[b];
  for (int t = 1; t <= H; ++t) {
    const double* lo = P.tube_lo + (static_cast<size_t>(b) * (H + 1) + t) * n;
    const double* hi = P.tube_hi + (static_cast<size_t>(b) * (H + 1) + t) * n;
    bool box_ok = t < nb;
    if (box_ok)
      for (int d = 0; d < n; ++d)
        if (!(finite(lo[d]) && finite(hi[d]))) box_ok = false;
    if (box_ok) {
      for (int c = 0; c < P.n_con; ++c) {
        const double g = con_margin(P, P.con[c], lo, hi);
        const double ng = -g;
        obj = add(obj, mul(P.penalty, (0.0 < ng) ? ng : 0.0));
      }
    } else if (P.n_con > 0) {
      obj = add(obj, mul(mul(P.penalty, P.diverged_margin), static_cast<double>(P.n_con)));
    }
  }
  P.objective[b] = obj;
  P.diverged[b] = P.status[b] != ST_OK ? 1 : 0;
}

// The objective's rollout part (nominal rollout + stage costs, mpc.hpp:170-184) with every W_l^T
// resident in shared memory for the whole launch (staged once per CTA, not per step and layer), up to
// 32 candidate warps per CTA persistent over the batch, and each lane's up-to-4 output units of a layer
// accumulated side by side (independent chains, each in the reference's j order) -- used whenever the
// network fits (C3: 157 KB).  It does not read the tube, so it runs concurrently with the tube kernel;
// plan_penalty_kernel then adds the constraint terms.  Together bit-identical to the above.
constexpr int kPlanMaxWarps = 32;
__global__ void __launch_bounds__(kPlanMaxWarps * 32) plan_rollout_resident_kernel(const PlanParams P, int vec,
                                                                                   int wtot) {
  extern __shared__ __align__(16) double psm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  const DevNet& N = P.net;
  const int n = P.n, m = P.m, H = P.H, L = N.L;
  int woff[kMaxLayers];
  {
    int off = 0;
    for (int l = 0; l < L; ++l) {
      const int rows = N.dims[l + 1], cols = N.dims[l];
      const double* wt = N.blob + N.wt_off[l];
      const int ld = N.ldt[l];
      for (int q = threadIdx.x; q < cols * rows; q += blockDim.x) {
        const int j = q / rows, oo = q % rows;
        psm[off + q] = __ldg(wt + static_cast<size_t>(j) * ld + oo);
      }
      woff[l] = off;
      off += cols * rows;
    }
  }
  __syncthreads();
  double* vin = psm + wtot + static_cast<size_t>(warp) * 2 * vec;
  double* vout = vin + vec;
  for (int b = blockIdx.x * nwarps + warp; b < P.B; b += gridDim.x * nwarps) {
    const double* acts = P.actions + static_cast<size_t>(b) * H * m;
    double x_reg = (lane < n) ? P.x0[lane] : 0.0;
    double obj = 0.0;
    for (int t = 0; t < H; ++t) {
      const double* u = acts + static_cast<size_t>(t) * m;
      __syncwarp();
      if (lane < n) vin[lane] = x_reg;
      for (int j = lane; j < m; j += 32) vin[n + j] = u[j];
      __syncwarp();
      double* a = vin;
      double* o = vout;
      for (int l = 0; l < L; ++l) {
        const int rows = N.dims[l + 1], cols = N.dims[l];
        const double* wsm = psm + woff[l];
        const double* bias = N.blob + N.b_off[l];
        const int act = N.acts[l];
        for (int o0 = lane; o0 < rows; o0 += 128) {
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          for (int j = 0; j < cols; ++j) {
            const double aj = a[j];
            const double* wr = wsm + j * rows + o0;
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (o0 + 32 * r < rows) acc[r] = add(acc[r], mul(wr[32 * r], aj));
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int oo = o0 + 32 * r;
            if (oo < rows) {
              double v = add(acc[r], __ldg(bias + oo));
              if (act == 0) v = (v < 0.0) ? 0.0 : v;  // MLPNet::h_relu (neural.hpp:85-87)
              else if (act == 1) v = tanh(v);
              o[oo] = v;
            }
          }
        }
        __syncwarp();
        double* tmp = a;
        a = o;
        o = tmp;
      }
      if (lane < n) x_reg = a[lane];
      if (lane == 0) {  // stage costs (mpc.hpp:171-183)
        for (int j = 0; j < m; ++j) obj = add(obj, mul(mul(P.r_w[j], u[j]), u[j]));
        for (int j = 0; j < n; ++j) {
          const double d = sub(a[j], P.x_goal[j]);
          obj = add(obj, mul(mul(P.q_w[j], d), d));
        }
      }
    }
    if (lane == 0) P.objective[b] = obj;  // rollout terms; plan_penalty_kernel adds the constraint terms
  }
}

// Constraint penalties over the certified tube (mpc.hpp:187-200), one thread per candidate, added to the
// rollout terms plan_rollout_resident_kernel left in P.objective.
__global__ void plan_penalty_kernel(const PlanParams P) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B) return;
  const int n = P.n, H = P.H;
  double obj = P.objective[b];
  const int nb = P.n_boxes[b];
  for (int t = 1; t <= H; ++t) {
    const double* lo = P.tube_lo + (static_cast<size_t>(b) * (H + 1) + t) * n;
    const double* hi = P.tube_hi + (static_cast<size_t>(b) * (H + 1) + t) * n;
    bool box_ok = t < nb;
    if (box_ok)
      for (int d = 0; d < n; ++d)
        if (!(finite(lo[d]) && finite(hi[d]))) box_ok = false;
    if (box_ok) {
      for (int c = 0; c < P.n_con; ++c) {
        const double g = con_margin(P, P.con[c], lo, hi);
        const double ng = -g;
        obj = add(obj, mul(P.penalty, (0.0 < ng) ? ng : 0.0));
      }
    } else if (P.n_con > 0) {
      obj = add(obj, mul(mul(P.penalty, P.diverged_margin), static_cast<double>(P.n_con)));
    }
  }
  P.objective[b] = obj;
  P.diverged[b] = P.status[b] != ST_OK ? 1 : 0;
}

// plan_step_margin (mpc.hpp:211-215) of K boxes: min over the constraints of
// Constraint::margin, folded with std::min's (b < a ? b : a) from +inf.
__global__ void box_margin_kernel(const PlanParams P, const double* lo, const double* hi, int K, double* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double worst = __longlong_as_double(0x7ff0000000000000ll);
  for (int c = 0; c < P.n_con; ++c) {
    const double g = con_margin(P, P.con[c], lo + static_cast<size_t>(k) * P.n, hi + static_cast<size_t>(k) * P.n);
    worst = (g < worst) ? g : worst;
  }
  out[k] = worst;
}

// MLPNet::forward (neural.hpp:58-76) of one input [x; u] -> x_next: the model
// as the simulator of mpc_run (the CLI's sim, reach_cli.cpp:445-449).  One
// CTA; thread o owns output o of each layer, dot product in matvec's order.
__global__ void model_step_kernel(const DevNet N, const double* xu, double* out, int maxw) {
  extern __shared__ __align__(16) double fwd[];
  double* a = fwd;
  double* o = fwd + maxw;
  for (int j = threadIdx.x; j < N.dims[0]; j += blockDim.x) a[j] = xu[j];
  __syncthreads();
  for (int l = 0; l < N.L; ++l) {
    const int rows = N.dims[l + 1], cols = N.dims[l];
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      const double* w = N.blob + N.w_off[l] + static_cast<size_t>(r) * N.ldw[l];
      double acc = 0.0;
      for (int j = 0; j < cols; ++j) acc = add(acc, mul(w[j], a[j]));
      double v = add(acc, N.blob[N.b_off[l] + r]);
      if (N.acts[l] == 0) v = (v < 0.0) ? 0.0 : v;
      else if (N.acts[l] == 1) v = tanh(v);
      o[r] = v;
    }
    __syncthreads();
    double* t = a;
    a = o;
    o = t;
  }
  for (int j = threadIdx.x; j < N.dims[N.L]; j += blockDim.x) out[j] = a[j];
}

// dt_interval_baseline (dt_reach.hpp:129-149): per step, freeze_trailing_inputs (neural.hpp:398-413)
// then interval_forward (neural.hpp:261-272: box_affine_image, + bias, act_interval) of the box; the
// naive tightness baseline.  One warp per sample; lane o owns output rows o, o + 32, ... of a layer,
// each a sequential iv_add(iv_scale) chain over the inputs as the reference's.
struct IBLArgs {
  DevNet net;
  int B, H, n, m, maxw;
  const double* x0_lo;    // [B][n]
  const double* x0_hi;
  const double* actions;  // [B][H][m] (or [H][m] shared)
  int actions_shared;
  double* out_lo;         // [B][H+1][n]
  double* out_hi;
  int* n_boxes;
  int* failed_step;
  int* status;
};

constexpr int kIblWarps = 8;

__global__ void __launch_bounds__(kIblWarps * 32) interval_baseline_kernel(const IBLArgs A) {
  extern __shared__ __align__(16) double ibl[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kIblWarps + warp;
  if (b >= A.B) return;
  const DevNet& N = A.net;
  const int n = A.n, m = A.m, W = A.maxw;
  double* lo0 = ibl + static_cast<size_t>(warp) * 4 * W;  // ping-pong boxes + the frozen first-layer bias
  double* hi0 = lo0 + W;
  double* lo1 = hi0 + W;
  double* hi1 = lo1 + W;
  double* bf = ibl + static_cast<size_t>(kIblWarps) * 4 * W + static_cast<size_t>(warp) * W;
  const double* acts = A.actions + (A.actions_shared ? 0 : static_cast<size_t>(b) * A.H * m);
  double* olo = A.out_lo + static_cast<size_t>(b) * (A.H + 1) * n;
  double* ohi = A.out_hi + static_cast<size_t>(b) * (A.H + 1) * n;
  for (int i = lane; i < n; i += 32) {
    lo0[i] = A.x0_lo[static_cast<size_t>(b) * n + i];
    hi0[i] = A.x0_hi[static_cast<size_t>(b) * n + i];
    olo[i] = lo0[i];
    ohi[i] = hi0[i];
  }
  __syncwarp();
  int nb = 1, fs = -1, st = 0;
  for (int k = 0; k < A.H; ++k) {
    // freeze_trailing_inputs: b'_i = b_i + sum_j W(i, n + j) u_j (j ascending)
    const double* u = acts + static_cast<size_t>(k) * m;
    for (int i = lane; i < N.dims[1]; i += 32) {
      const double* w = N.blob + N.w_off[0] + static_cast<size_t>(i) * N.ldw[0];
      double bi = N.blob[N.b_off[0] + i];
      for (int j = 0; j < m; ++j) bi = add(bi, mul(w[n + j], u[j]));
      bf[i] = bi;
    }
    __syncwarp();
    double *hl = lo0, *hh = hi0, *ol = lo1, *oh = hi1;
    for (int l = 0; l < N.L; ++l) {
      const int rows = N.dims[l + 1], cols = (l == 0) ? n : N.dims[l];
      const int act = N.acts[l];
      for (int i = lane; i < rows; i += 32) {
        const double* w = N.blob + N.w_off[l] + static_cast<size_t>(i) * N.ldw[l];
        double al = 0.0, ah = 0.0;  // box_affine_image: acc = iv_add(acc, iv_scale(W(i, j), x_j))
        for (int j = 0; j < cols; ++j) {
          const double a = w[j];
          const bool pos = a >= 0.0;
          al = add(al, mul(a, pos ? hl[j] : hh[j]));
          ah = add(ah, mul(a, pos ? hh[j] : hl[j]));
        }
        const double bb = (l == 0) ? bf[i] : N.blob[N.b_off[l] + i];
        double pl = add(al, bb), ph = add(ah, bb);  // iv_add(p, [b, b])
        if (act == 0) {  // act_interval: std::max(x, 0.0)
          pl = (pl < 0.0) ? 0.0 : pl;
          ph = (ph < 0.0) ? 0.0 : ph;
        } else if (act == 1) {
          pl = tanh(pl);
          ph = tanh(ph);
        }
        ol[i] = pl;
        oh[i] = ph;
      }
      __syncwarp();
      double* t0 = hl;
      double* t1 = hh;
      hl = ol;
      hh = oh;
      ol = t0;
      oh = t1;
    }
    bool fin = true;
    for (int i = lane; i < n; i += 32) {
      olo[static_cast<size_t>(k + 1) * n + i] = hl[i];
      ohi[static_cast<size_t>(k + 1) * n + i] = hh[i];
      fin = fin && finite(hl[i]) && finite(hh[i]);
    }
    fin = __all_sync(0xffffffffu, fin);
    nb = k + 2;
    if (!fin) {  // tube.mark_failed(k, "diverged box")
      fs = k;
      st = 3;
      break;
    }
    if (hl != lo0) {  // keep the box in the (lo0, hi0) slot for the next step
      for (int i = lane; i < n; i += 32) {
        lo0[i] = hl[i];
        hi0[i] = hh[i];
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    A.n_boxes[b] = nb;
    A.failed_step[b] = fs;
    A.status[b] = st;
  }
}

}  // namespace rb
