// Internal (not ABI): host helpers of the tensor-core contraction shared by the
// library's translation units.
#pragma once

#include <cuda.h>

#include <cstdint>

struct reach_ctx;

namespace rbh {
// TMA tensor map over split int8 operand planes [slices][Mp][Kp] with
// {128 B, 128 rows, 1 slice} boxes and the 128-byte swizzle.
int make_slice_tmap(reach_ctx* ctx, CUtensorMap* map, const int8_t* planes, int Mp, int Kp, int slices);
}  // namespace rbh
