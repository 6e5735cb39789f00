// Kernel-parameter types of the tensor-core wide kernel (tcw_kernel.cuh), shared
// with the host planner (reach_capi.cu) without pulling in the kernel.
#pragma once

#include <cuda.h>

#include "dt_kernel.cuh"

namespace rb {

struct OzNet {
  const CUtensorMap* tmap;  // [kMaxLayers] TMA maps over the split planes of W_l^T
  const int* ea;            // A-row scale exponents of layer l at e_off[l]
  const double* l1a;        // A-row L1 norms
  long long e_off[kMaxLayers];
  int mp[kMaxLayers];       // padded rows of W_l^T (= dims[l]) and K (= dims[l+1])
  int kp[kMaxLayers];
};

struct TcwParams {
  OzNet net, ctl;
  int o_relax, o_misc, o_int, o_bar;  // shared-memory byte offsets (after the 1024-aligned U0 region)
};

}  // namespace rb
