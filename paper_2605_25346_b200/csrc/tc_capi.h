// Internal (not ABI): host helpers of the tensor-core contraction shared by the
// library's translation units.
#pragma once

#include <cuda.h>

#include <cstdint>

#include "tcw_types.cuh"

struct reach_ctx;
struct reach_net;

namespace rbh {
// Plans the tensor-core wide kernel on top of plan_wide's layout (state buffers, hw):
// builds the nets' split planes on first use, sets the shared-memory offsets, smem
// bytes and grid.  Returns a reach_status.
int plan_tcw(reach_ctx* ctx, const reach_net* net, const reach_net* ctl, int n, long long B, rb::DTParams& P,
             size_t& smem, int& grid, rb::TcwParams& X);
cudaError_t tcw_launch(const rb::DTParams& P, const rb::TcwParams& X, size_t smem, int grid, cudaStream_t s);
// Frees a net's tensor-core planes (reach_net_free).
void free_oz(reach_net* net);
// TMA tensor map over split int8 operand planes [slices][Mp][Kp] with
// {128 B, 128 rows, 1 slice} boxes and the 128-byte swizzle.
int make_slice_tmap(reach_ctx* ctx, CUtensorMap* map, const int8_t* planes, int Mp, int Kp, int slices);
}  // namespace rbh
