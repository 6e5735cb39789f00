// Dependent-chain latencies on sm_100a (one warp): DADD, DFMA, DMUL, DDIV (__ddiv_rn), SHFL of a double,
// LDS.64, and a shuffle-xor max round of the fold's pivot search.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane;
  sm[lane + 32] = lane;
  __syncwarp();
  double x = 1.0 + lane * 1e-9, y = 1.000001;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, 1e-12);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dmul_rn(x, y);
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ddiv_rn(x, y);
  t1 = clock64();
  cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  cyc[4] = t1 - t0;
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = static_cast<int>(sm[idx & 63]) + (i & 1);
  t1 = clock64();
  cyc[5] = t1 - t0;
  double bv = x;
  int bi = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    bv += 1e-300;
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[lane] = x + idx + bv + bi;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 64 * 8);
  cudaMalloc(&c, 16 * 8);
  const int iters = 4096;
  chains<<<1, 32>>>(d, c, iters);
  chains<<<1, 32>>>(d, c, iters);
  long long h[16];
  cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DADD", "DFMA", "DMUL", "DDIV(__ddiv_rn)", "SHFL double", "LDS (dependent)", "argmax 5 rounds"};
  for (int i = 0; i < 7; ++i) printf("%-18s %8.1f cycles/op\n", nm[i], double(h[i]) / iters);
  return 0;
}
