// Pipeline P2P channels: IPC-mapped receive rings, copy-engine transfers,
// stream memory-op flags.  See p2p.h for the protocol.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.h"
#include "p2p.h"
#include "runtime.h"

namespace mp {

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static WaitValueFn g_wait = nullptr;
static WriteValueFn g_write = nullptr;

static mp_status load_memops() {
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait = reinterpret_cast<WaitValueFn>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_write = reinterpret_cast<WriteValueFn>(p);
    ok = g_wait && g_write;
  });
  return ok ? MP_OK : set_err(MP_ECUDA, "stream memory operations unavailable");
}

static inline size_t al(size_t x) { return (x + 4095) & ~size_t(4095); }

// slab layout
static size_t ring_bytes(size_t slot) { return al(slot) * P2P_SLOTS; }
static char* act_ring(void* slab, size_t slot) { return (char*)slab; }
static char* grad_ring(void* slab, size_t slot) { return (char*)slab + ring_bytes(slot); }
static uint32_t* flags(void* slab, size_t slot) { return (uint32_t*)((char*)slab + 2 * ring_bytes(slot)); }
// flag indices
static inline int F_ACT_FULL(int k) { return k; }
static inline int F_GRAD_FULL(int k) { return P2P_SLOTS + k; }
static inline int F_ACT_EMPTY(int k) { return 2 * P2P_SLOTS + k; }
static inline int F_GRAD_EMPTY(int k) { return 3 * P2P_SLOTS + k; }

static mp_status cu(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) return set_err(MP_ECUDA, "%s failed (CUresult %d)", what, (int)r);
  return MP_OK;
}

mp_status p2p_release(mp_ctx* c) {
  P2PRing& R = c->p2p;
  if (R.prev_slab) cudaIpcCloseMemHandle(R.prev_slab);
  if (R.next_slab && R.next_slab != R.prev_slab) cudaIpcCloseMemHandle(R.next_slab);
  if (R.slab) cudaFree(R.slab);
  R = P2PRing{};
  return MP_OK;
}

mp_status p2p_ensure(mp_ctx* c, size_t slot_bytes) {
  if (c->p == 1) return MP_OK;
  P2PRing& R = c->p2p;
  if (R.slab && R.slot_bytes >= slot_bytes) return MP_OK;
  MP_TRY(load_memops());
  // collective over the world: every rank calls run_batch with the same b
  MP_CUDA(cudaDeviceSynchronize());
  p2p_release(c);
  const size_t total = 2 * ring_bytes(slot_bytes) + 4096;
  MP_CUDA(cudaMalloc(&R.slab, total));
  MP_CUDA(cudaMemset(flags(R.slab, slot_bytes), 0, 4096));
  R.slot_bytes = slot_bytes;
  cudaIpcMemHandle_t h;
  MP_CUDA(cudaIpcGetMemHandle(&h, R.slab));
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  char *dsend = nullptr, *drecv = nullptr;
  MP_CUDA(cudaMalloc(&dsend, hb));
  MP_CUDA(cudaMalloc(&drecv, hb * c->world));
  MP_CUDA(cudaMemcpy(dsend, &h, hb, cudaMemcpyHostToDevice));
  ncclResult_t r = ncclAllGather(dsend, drecv, hb, ncclUint8, c->world_comm, c->cs);
  if (r != ncclSuccess) return set_err(MP_ENCCL, "ipc handle all-gather: %s", ncclGetErrorString(r));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  std::vector<char> all(hb * c->world);
  MP_CUDA(cudaMemcpy(all.data(), drecv, all.size(), cudaMemcpyDeviceToHost));
  cudaFree(dsend);
  cudaFree(drecv);
  const int dp_base = (c->rank / (c->t * c->p)) * c->t * c->p;
  const int prev_rank = dp_base + ((c->pp - 1 + c->p) % c->p) * c->t + c->tp;
  const int next_rank = dp_base + ((c->pp + 1) % c->p) * c->t + c->tp;
  cudaIpcMemHandle_t hp, hn;
  memcpy(&hp, all.data() + hb * prev_rank, hb);
  memcpy(&hn, all.data() + hb * next_rank, hb);
  MP_CUDA(cudaIpcOpenMemHandle(&R.prev_slab, hp, cudaIpcMemLazyEnablePeerAccess));
  if (next_rank == prev_rank) R.next_slab = R.prev_slab;
  else MP_CUDA(cudaIpcOpenMemHandle(&R.next_slab, hn, cudaIpcMemLazyEnablePeerAccess));
  int flush = 0;
  cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, c->device);
  R.flush_ok = flush != 0;
  R.n_act_sent = R.n_act_recv = R.n_grad_sent = R.n_grad_recv = 0;
  // every rank has zeroed its flags before anyone may write into them
  MP_CUDA(cudaDeviceSynchronize());
  r = ncclAllReduce(c->d_loss + 40, c->d_loss + 40, 1, ncclFloat32, ncclSum, c->world_comm, c->cs);
  if (r != ncclSuccess) return set_err(MP_ENCCL, "p2p setup barrier: %s", ncclGetErrorString(r));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  return MP_OK;
}

static mp_status send(mp_ctx* c, bool act, const void* src, size_t bytes, cudaStream_t st) {
  P2PRing& R = c->p2p;
  if (!R.slab || bytes > R.slot_bytes) return set_err(MP_ESTATE, "p2p ring not set up");
  uint64_t& n = act ? R.n_act_sent : R.n_grad_sent;
  const int k = (int)(n % P2P_SLOTS);
  const uint32_t lap = (uint32_t)(n / P2P_SLOTS);
  void* peer = act ? R.next_slab : R.prev_slab;
  uint32_t* my_flags = flags(R.slab, R.slot_bytes);
  uint32_t* peer_flags = flags(peer, R.slot_bytes);
  const int fe = act ? F_ACT_EMPTY(k) : F_GRAD_EMPTY(k);
  const int ff = act ? F_ACT_FULL(k) : F_GRAD_FULL(k);
  char* dst = (act ? act_ring(peer, R.slot_bytes) : grad_ring(peer, R.slot_bytes)) + (size_t)k * al(R.slot_bytes);
  // the receiver released this slot's previous lap
  MP_TRY(cu(g_wait((CUstream)st, (CUdeviceptr)(my_flags + fe), lap, CU_STREAM_WAIT_VALUE_GEQ), "wait empty"));
  MP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  MP_TRY(cu(g_write((CUstream)st, (CUdeviceptr)(peer_flags + ff), lap + 1, CU_STREAM_WRITE_VALUE_DEFAULT),
            "write full"));
  ++n;
  return MP_OK;
}

// slot -> destination copy on the consuming stream (16-byte vectors, grid sized to the SMs)
__global__ void slot_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

static mp_status recv(mp_ctx* c, bool act, void* dst, size_t bytes, cudaStream_t st) {
  P2PRing& R = c->p2p;
  if (!R.slab || bytes > R.slot_bytes) return set_err(MP_ESTATE, "p2p ring not set up");
  uint64_t& n = act ? R.n_act_recv : R.n_grad_recv;
  const int k = (int)(n % P2P_SLOTS);
  const uint32_t lap = (uint32_t)(n / P2P_SLOTS);
  void* peer = act ? R.prev_slab : R.next_slab;      // the sender
  uint32_t* my_flags = flags(R.slab, R.slot_bytes);
  uint32_t* peer_flags = flags(peer, R.slot_bytes);
  const int ff = act ? F_ACT_FULL(k) : F_GRAD_FULL(k);
  const int fe = act ? F_ACT_EMPTY(k) : F_GRAD_EMPTY(k);
  const char* src = (act ? act_ring(R.slab, R.slot_bytes) : grad_ring(R.slab, R.slot_bytes)) + (size_t)k * al(R.slot_bytes);
  unsigned wflags = CU_STREAM_WAIT_VALUE_GEQ | (R.flush_ok ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
  MP_TRY(cu(g_wait((CUstream)st, (CUdeviceptr)(my_flags + ff), lap + 1, wflags), "wait full"));
  if (bytes % 16 == 0 && ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n16 = bytes / 16;
    const int grid = (int)std::min<size_t>((n16 + 255) / 256, (size_t)num_sms() * 4);
    slot_copy_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), n16);
    count_launch();
    MP_CUDA(cudaGetLastError());
  } else {
    MP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  }
  MP_TRY(cu(g_write((CUstream)st, (CUdeviceptr)(peer_flags + fe), lap + 1, CU_STREAM_WRITE_VALUE_DEFAULT),
            "write empty"));
  ++n;
  return MP_OK;
}

mp_status p2p_send_act(mp_ctx* c, const void* src, size_t bytes, cudaStream_t st) { return send(c, true, src, bytes, st); }
mp_status p2p_send_grad(mp_ctx* c, const void* src, size_t bytes, cudaStream_t st) { return send(c, false, src, bytes, st); }
mp_status p2p_recv_act(mp_ctx* c, void* dst, size_t bytes, cudaStream_t st) { return recv(c, true, dst, bytes, st); }
mp_status p2p_recv_grad(mp_ctx* c, void* dst, size_t bytes, cudaStream_t st) { return recv(c, false, dst, bytes, st); }

}  // namespace mp
