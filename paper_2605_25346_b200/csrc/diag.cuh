// FP64 pipe microbenchmarks (roofline denominators).  MEASURED_PEAKS.json only
// carries HBM and bf16 tensor peaks; the DT kernels are FP64-pipe bound, so
// bench.py measures the FP64 ceilings on the same box with these kernels.
#pragma once

#include <cuda_runtime.h>

namespace rb {

// 16 independent DFMA chains per thread: 2 flops per instruction.
__global__ void __launch_bounds__(256) fp64_fma_peak_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;  // keep the work alive
}

// DMUL + DADD pairs (the exact kernels' instruction mix): 1 flop per instruction.
__global__ void __launch_bounds__(256) fp64_muladd_peak_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __dadd_rn(__dmul_rn(x[i], a), b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

}  // namespace rb
