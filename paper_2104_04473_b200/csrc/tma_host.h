// Host-side TMA tensor-map construction (gemm.cu).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace mp {
// 3-D tensor map: dims (inner, outer, batch) with element strides (ld, batch_stride),
// 128-byte swizzle, box (128 B of inner, box_outer, 1); esize 2 = bf16, 4 = fp32.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t batch,
              uint64_t ld_elems, uint64_t batch_stride_elems, uint32_t box_outer, int esize = 2);
}  // namespace mp
