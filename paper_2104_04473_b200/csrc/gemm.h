// Internal entry points of the GEMM engine (gemm.cu) used by the layer code.
#pragma once
#include <cuda_runtime.h>

#include "../../include/mp_ops.h"

namespace mp {

// Cross-entropy statistics epilogue of the logit GEMM (a18): with a
// GemmCe the bf16 GEMM also writes, per (row, column block, epilogue half),
// the fp32 (max, sum exp(x - max)) of the unrounded logits to part
// [M][2 gemm_ce_nblocks(g)] and the fp32 logit of the row's label (if in this
// shard: lab[beta * lab_ld + i] - v0 in [0, N)) to tgt[row].
struct GemmCe {
  float2* part;
  float* tgt;
  const int* lab;
  int lab_ld, b, v0;
};

mp_status gemm(mp_dtype dt, const mp_gemm_desc& g, cudaStream_t st, const GemmCe* ce = nullptr);
int gemm_ce_nblocks(const mp_gemm_desc& g);
void gemm_set_max_ctas(int n);

}  // namespace mp
