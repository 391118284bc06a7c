// Layer / model-end building blocks used by the runtime (layer.cu).
#pragma once
#include "runtime.h"

namespace mp {

mp_status nccl_check(ncclResult_t r, const char* what);
mp_status alloc_async(mp_ctx* c, void** p, size_t bytes, cudaStream_t st);
mp_status ensure_workspace(mp_ctx* c, int b);
mp_status layer_fwd(mp_ctx* c, int layer, int b, const void* x, void* y, LayerStash& st);
mp_status layer_bwd(mp_ctx* c, int layer, const LayerStash& st, const void* dy, void* dx);
mp_status stash_release(mp_ctx* c, LayerStash& st, cudaStream_t s);
mp_status embed_forward(mp_ctx* c, const int* dtok, int tok_ld, int b, void* X);
mp_status embed_backward(mp_ctx* c, const int* dtok, int tok_ld, int b, const void* dX);
// defer_slot >= 0 (bf16): dlogits and Z of this microbatch go to row block defer_slot of
// c->head_dl / c->head_z and the dE GEMM is left to head_dE_deferred at the flush.
mp_status head_fwd_bwd(mp_ctx* c, const void* X, const int* dlab, int lab_ld, int b, float scale, void* dX,
                       int defer_slot = -1);
// seconds per fused g / f reduction of s*b*h elements on the NVLS path (collective over TP)
mp_status tp_reduce_probe(mp_ctx* c, int b, int iters, double* seconds);
// dE_r += dlogits^T Z over the first n_slots row blocks of b*s rows (one GEMM, K = n_slots b s)
mp_status head_dE_deferred(mp_ctx* c, int b, int n_slots);

}  // namespace mp
