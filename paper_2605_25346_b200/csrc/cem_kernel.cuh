// plan_cem's sampler on the device (mpc.hpp:258-335): candidate generation from the
// reference's normal stream, the stable sort of the scores, incumbent retention and
// the smoothed elite refit -- in the reference's floating-point order (separate
// roundings, IEEE division / sqrt), so the whole replan stays bit-identical to the
// host loop while the population, the scores and the CEM state never leave HBM.
// The normals themselves come from the host (std::mt19937_64 + glibc's log / sin /
// cos, rng.hpp:24-37: bit-identical only there); they are uploaded once per
// iteration, ahead of use.
#pragma once

#include "dt_common.cuh"

namespace rb {
namespace cem {

struct CemDev {
  double* cand;         // [pop][dim] candidate population
  const double* z;      // normals of the iteration being generated, in stream order (row 0 skipped when it > 0)
  const double* score;  // [pop] objectives of the evaluated population
  const int* div;       // [pop] diverged flags
  double* mean;         // [dim]
  double* stdv;         // [dim]
  double* best;         // [dim] incumbent
  double* best_obj;     // [1]
  int* any_finite;      // [1]
  double* hist;         // [iterations]
  const double* lo;     // [m] action box
  const double* hi;
  int pop, dim, m, n_elite;
  double smoothing;
};

// std::clamp(v, lo, hi)
__device__ __forceinline__ double clampd(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// Candidates of iteration `it` (mpc.hpp:290-299): row 0 is the incumbent after the first iteration,
// every other entry mean + std * z, clipped to the action box.
__global__ void cem_generate_kernel(CemDev S, int it) {
  const long long zskip = it > 0 ? S.dim : 0;  // the incumbent row draws no normals
  const long long total = static_cast<long long>(S.pop) * S.dim;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e / S.dim), q = static_cast<int>(e - static_cast<long long>(k) * S.dim);
    double v;
    if (it > 0 && k == 0) {
      v = S.best[q];
    } else {
      const int j = q % S.m;
      v = clampd(add(S.mean[q], mul(S.stdv[q], S.z[e - zskip])), S.lo[j], S.hi[j]);
    }
    S.cand[e] = v;
  }
}

// Initial state (mpc.hpp:276-281): mean = box centre, std = init_std, best = clip(mean).
__global__ void cem_init_kernel(CemDev S, double init_std) {
  for (int q = threadIdx.x; q < S.dim; q += blockDim.x) {
    const int j = q % S.m;
    const double c = mul(0.5, add(S.lo[j], S.hi[j]));
    S.mean[q] = c;
    S.stdv[q] = init_std;
    S.best[q] = clampd(c, S.lo[j], S.hi[j]);
  }
  if (threadIdx.x == 0) {
    *S.best_obj = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    *S.any_finite = 0;
  }
}

// Bitonic sort of (order key of the score, index) pairs: the same permutation as std::stable_sort by
// score (ties keep index order; -0 and +0 compare equal as in operator<).  One CTA; smem keys.
__device__ __forceinline__ void cx(unsigned long long* key, int* idx, int a, int b, bool up) {
  const unsigned long long ka = key[a], kb = key[b];
  const int ia = idx[a], ib = idx[b];
  const bool gt = (ka > kb) || (ka == kb && ia > ib);
  if (gt == up) {
    key[a] = kb;
    key[b] = ka;
    idx[a] = ib;
    idx[b] = ia;
  }
}

// Sort, incumbent, history and the smoothed refit of iteration `it` (mpc.hpp:300-333).
__global__ void cem_update_kernel(CemDev S, int it, int p2) {
  extern __shared__ unsigned long long csm[];
  unsigned long long* key = csm;
  int* idx = reinterpret_cast<int*>(key + p2);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = tid; k < p2; k += nt) {
    if (k < S.pop) {
      double s = S.score[k];
      if (s == 0.0) s = 0.0;  // -0 == +0 under operator<
      key[k] = order_key(s);
      idx[k] = k;
    } else {
      key[k] = ~0ull;
      idx[k] = 0x7fffffff;
    }
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < p2 / 2; t += nt) {
        const int a = 2 * stride * (t / stride) + (t % stride), b = a + stride;
        const bool up = ((a & size) == 0);
        cx(key, idx, a, b, up);
      }
      __syncthreads();
    }
  }
  const int top = idx[0];
  __shared__ int improve;
  if (tid == 0) {
    const double st = S.score[top];
    double bo = *S.best_obj;
    improve = st < bo;
    if (improve) {
      bo = st;
      *S.best_obj = st;
    }
    int any = *S.any_finite;
    for (int e = 0; e < S.n_elite; ++e)
      if (!S.div[idx[e]]) any = 1;
    *S.any_finite = any;
    S.hist[it] = bo;
  }
  __syncthreads();
  if (improve)
    for (int q = tid; q < S.dim; q += nt) S.best[q] = S.cand[static_cast<long long>(top) * S.dim + q];
  const double sm = S.smoothing, ne = static_cast<double>(S.n_elite);
  for (int q = tid; q < S.dim; q += nt) {
    double em = 0.0;
    for (int e = 0; e < S.n_elite; ++e) em = add(em, S.cand[static_cast<long long>(idx[e]) * S.dim + q]);
    em = __ddiv_rn(em, ne);
    double ev = 0.0;
    for (int e = 0; e < S.n_elite; ++e) {
      const double d = sub(S.cand[static_cast<long long>(idx[e]) * S.dim + q], em);
      ev = add(ev, mul(d, d));
    }
    const double es = __dsqrt_rn(__ddiv_rn(ev, ne));
    S.mean[q] = add(mul(sm, S.mean[q]), mul(sub(1.0, sm), em));
    const double v = add(mul(sm, S.stdv[q]), mul(sub(1.0, sm), es));
    S.stdv[q] = (1e-6 < v) ? v : 1e-6;  // std::max(1e-6, v)
  }
}

// Multi-GPU: every rank's padded slice of scores / diverged flags back into candidate order.
__global__ void cem_unpad_kernel(const double* gs, const int* gd, int world, int width, int pop, double* score,
                                 int* div) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < pop; k += gridDim.x * blockDim.x) {
    const int base = pop / world, rem = pop % world;
    // rank r owns [r base + min(r, rem), ... + base + (r < rem))
    int r = (rem > 0 && k < rem * (base + 1)) ? k / (base + 1) : (base > 0 ? rem + (k - rem * (base + 1)) / base : 0);
    const int r0 = r * base + min(r, rem);
    score[k] = gs[static_cast<long long>(r) * width + (k - r0)];
    div[k] = gd[static_cast<long long>(r) * width + (k - r0)];
  }
}

}  // namespace cem
}  // namespace rb
