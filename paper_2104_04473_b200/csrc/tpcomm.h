// TP-symmetric buffers for the fused g / f all-reduce.
// The row-parallel GEMM (proj, FC2) and the dgrad GEMMs that feed a
// LayerNorm backward write their partial products into one of two buffers of
// a window registered with NCCL as symmetric memory; after a one-thread
// NVLS barrier the consuming elementwise kernel reads the multicast address
// with multimem.ld_reduce, so the NVSwitch sums the t partials during the
// load and no separate all-reduce pass runs.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstddef>
#include <cstdint>

#include "../../include/mp.h"

struct mp_ctx;

namespace mp {

struct TpSym {
  bool tried = false;        // setup attempted for the current size
  bool on = false;           // NVLS path active
  size_t buf_bytes = 0;      // bytes per buffer
  void* base = nullptr;      // local view of the window
  char* mc = nullptr;        // multicast view of the window
  ncclWindow_t win = nullptr;
  void* devcomm = nullptr;   // ncclDevComm (opaque here)
  uint32_t epoch = 0;        // barriers issued
  unsigned long long next = 0;  // buffers handed out
};

// (Re)allocates the symmetric buffers for `buf_bytes` per buffer when the TP
// path is NVLS (collective over the TP group; call on every TP rank in the
// same order).  Leaves tps.on = false when multicast is unavailable and the
// configuration allows the NCCL fallback.
mp_status tp_sym_ensure(mp_ctx* c, size_t buf_bytes);
// Next buffer: local pointer for the producer, multicast pointer for the consumer.
void tp_sym_next(mp_ctx* c, void** local, const void** mc);
// Two-shot variant (t >= 4 by default; MP_TP_NVLS_SHOT=1|2 overrides): after
// the barrier, every rank reduce-loads only its 1/t slab of the partial sums
// and multicast-stores the sum into the landing buffer paired with the last
// buffer handed out; after a second barrier every rank holds the full sum in
// its local copy (returned in *out).  NVLink egress per GPU ~ (1 + 1/t) x the
// tensor instead of t x (one-shot).
bool tp_sym_two_shot(const mp_ctx* c);
mp_status tp_sym_reduce_two_shot(mp_ctx* c, size_t n_elems, cudaStream_t st, const void** out);
// All TP ranks' partials written (every prior kernel of this stream on every rank done).
mp_status tp_sym_barrier(mp_ctx* c, cudaStream_t st);
void tp_sym_free(mp_ctx* c);
bool tp_sym_debug_local();

}  // namespace mp
