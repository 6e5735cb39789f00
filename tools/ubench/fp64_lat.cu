// FP64 latency / throughput microbenchmarks on sm_100a (one SM, controlled warp counts).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dadd_chain(double* out, int iters, long long* cyc) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  const double b = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = __dadd_rn(x[i], b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 1.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
  else if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
}

// the GEMM micro-kernel shape: 24 independent DMUL then 24 dependent DADD per "row"
__global__ void gemm_shape(double* out, int iters, long long* cyc) {
  double acc[24], t[24];
  double lam[6], w[4];
#pragma unroll
  for (int i = 0; i < 24; ++i) acc[i] = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i) lam[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = 0.5 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) t[i * 4 + c] = __dmul_rn(lam[i], w[c]);
#pragma unroll
    for (int q = 0; q < 24; ++q) acc[q] = __dadd_rn(acc[q], t[q]);
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __dadd_rn(w[i], 1e-12);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 24; ++i) s += acc[i];
  if (s == 1.5) out[0] = s;
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 64 + threadIdx.x / 32] = t1 - t0;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 64 * 8 * 148);
  long long h[64];
  const int iters = 4096;
  auto run = [&](const char* name, void (*k)(double*, int, long long*), int warps, double instr_per_iter) {
    k<<<1, warps * 32>>>(d, iters, c);
    cudaDeviceSynchronize();
    k<<<1, warps * 32>>>(d, iters, c);
    cudaMemcpy(h, c, 64 * 8, cudaMemcpyDeviceToHost);
    double cyc = (double)h[0];
    printf("%-22s warps=%2d  cycles/iter/warp=%7.2f  warp-instr/cycle/SM=%5.2f\n", name, warps, cyc / iters,
           warps * instr_per_iter * iters / cyc);
  };
  for (int w : {1, 2, 4, 8, 16}) run("dadd_chain ILP1", dadd_chain<1>, w, 1);
  for (int w : {1, 4, 8}) run("dadd_chain ILP4", dadd_chain<4>, w, 4);
  for (int w : {1, 4, 8, 16}) run("dadd_chain ILP16", dadd_chain<16>, w, 16);
  for (int w : {1, 4, 8, 12, 16}) run("gemm_shape (52 fp64)", gemm_shape, w, 52);
  return 0;
}
