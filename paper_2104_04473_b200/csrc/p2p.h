// Pipeline point-to-point channels over NVLink without SM-resident waits.
//
// Each directed channel (activations r -> r+1, gradients r+1 -> r) is a FIFO
// of K slots living in the RECEIVER's HBM (CUDA IPC-mapped into the sender).
// Message n uses slot n % K, lap n / K:
//   sender (channel stream): wait  empty[slot] >= lap        (stream memory op, local)
//                            copy  src -> peer slot          (copy engine over NVLink)
//                            write peer full[slot] = lap + 1 (stream memory op, remote)
//   receiver (the consuming compute stream, which needs the data next anyway):
//                            wait  full[slot] >= lap + 1     (local)
//                            copy  slot -> private buffer    (SM kernel, ~3 us for 9 MB)
//                            write peer empty[slot] = lap + 1 (remote, frees the slot)
// Waiting holds no SM.  A blocked send never stalls compute, and a receive
// waits only for the message the compute stream consumes next: the send
// order of every channel equals its consume order (FIFO matching is exact --
// checked against the oracle for every schedule), and the receiver has freed
// every earlier slot before it waits, so no wait cycle can form.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

struct mp_ctx;

namespace mp {

constexpr int P2P_SLOTS = 4;

struct P2PRing {
  void* slab = nullptr;          // local allocation: [act ring | grad ring | flags]
  size_t slot_bytes = 0;
  // peers' slabs mapped into this process (prev = pp-1, next = pp+1 mod p)
  void* prev_slab = nullptr;
  void* next_slab = nullptr;
  uint64_t n_act_sent = 0, n_act_recv = 0, n_grad_sent = 0, n_grad_recv = 0;
  bool flush_ok = false;
};

mp_status p2p_ensure(mp_ctx* c, size_t slot_bytes);
mp_status p2p_release(mp_ctx* c);
// Enqueue the transfer of `bytes` from `src` (on stream st) to the next / previous device.
mp_status p2p_send_act(mp_ctx* c, const void* src, size_t bytes, cudaStream_t st);
mp_status p2p_send_grad(mp_ctx* c, const void* src, size_t bytes, cudaStream_t st);
// Enqueue the reception into `dst` on stream st (dst owned by the caller).
mp_status p2p_recv_act(mp_ctx* c, void* dst, size_t bytes, cudaStream_t st);
mp_status p2p_recv_grad(mp_ctx* c, void* dst, size_t bytes, cudaStream_t st);

}  // namespace mp
