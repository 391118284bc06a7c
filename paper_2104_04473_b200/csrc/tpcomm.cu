// NVLS symmetric-memory plumbing of the fused TP all-reduce (see tpcomm.h).
// NCCL 2.28's symmetric windows provide the memory and the multicast mapping;
// the reduction itself happens in our elementwise kernels (multimem.ld_reduce),
// the barrier is ours (multimem.red on a counter in the window).
#include <cuda.h>
#include <nccl_device.h>

#include <cstdlib>
#include <string>
#include <algorithm>

#include "common.h"
#include "runtime.h"
#include "tpcomm.h"

namespace mp {

mp_status nccl_check(ncclResult_t r, const char* what);

static constexpr size_t FLAG_BYTES = 4096;   // barrier counter lives at the window's start

__global__ void tp_query_kernel(ncclWindow_t w, ncclDevComm dev, void** out) {
  out[0] = ncclGetLsaMultimemPointer(w, 0, dev);
  out[1] = ncclGetLocalPointer(w, 0);
}

// Arrive (multicast add: every rank's counter += 1), then wait until all t
// ranks have arrived for this epoch.  Bounded: a peer that never arrives traps
// after ~20 s instead of hanging the device.
__global__ void tp_barrier_kernel(uint32_t* mc_flag, const uint32_t* flag, uint32_t target) {
  if (threadIdx.x != 0) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], 1;" ::"l"(mc_flag) : "memory");
  const long long t0 = clock64();
  uint32_t v;
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - target) >= 0) break;
    if (clock64() - t0 > 40000000000LL) __trap();
  }
}

void tp_sym_free(mp_ctx* c) {
  TpSym& s = c->tps;
  if (s.devcomm) {
    ncclDevCommDestroy(c->tp_comm, reinterpret_cast<ncclDevComm*>(s.devcomm));
    delete reinterpret_cast<ncclDevComm*>(s.devcomm);
  }
  if (s.win) ncclCommWindowDeregister(c->tp_comm, s.win);
  if (s.base) ncclMemFree(s.base);
  s = TpSym{};
}

static bool want_nvls(const mp_ctx* c) {
  if (c->t <= 1) return false;
  if (c->cfg.tp_comm == MP_TP_COMM_NCCL) return false;
  const char* e = getenv("MP_TP_COMM");   // ablation override: "nccl" forces the paper's all-reduce
  if (e && std::string(e) == "nccl") return false;
  return true;
}

mp_status tp_sym_ensure(mp_ctx* c, size_t buf_bytes) {
  TpSym& s = c->tps;
  if (!want_nvls(c)) { s.tried = true; return MP_OK; }
  if (s.tried && s.buf_bytes >= buf_bytes) return MP_OK;
  MP_CUDA(cudaDeviceSynchronize());
  const bool required = c->cfg.tp_comm == MP_TP_COMM_NVLS;
  tp_sym_free(c);
  s.tried = true;
  buf_bytes = (buf_bytes + 4095) & ~size_t(4095);
  const size_t total = FLAG_BYTES + 4 * buf_bytes;   // 2 partial-sum buffers + 2 landing buffers
  int mc_ok = 0;
  {
    using attr_fn = CUresult (*)(int*, CUdevice_attribute, CUdevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && p)
      if (reinterpret_cast<attr_fn>(p)(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)c->device) !=
          CUDA_SUCCESS)
        mc_ok = 0;
  }
  // the decision must be identical on all TP ranks: agree on min(mc_ok)
  int* d_flag = nullptr;
  MP_CUDA(cudaMalloc(&d_flag, sizeof(int)));
  MP_CUDA(cudaMemcpy(d_flag, &mc_ok, sizeof(int), cudaMemcpyHostToDevice));
  MP_TRY(nccl_check(ncclAllReduce(d_flag, d_flag, 1, ncclInt32, ncclMin, c->tp_comm, c->cs), "nvls probe"));
  MP_CUDA(cudaMemcpyAsync(&mc_ok, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->cs));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  cudaFree(d_flag);
  if (!mc_ok) {
    if (required) return set_err(MP_EUNSUPPORTED, "tp_comm = NVLS but multicast is not supported on this device");
    return MP_OK;
  }
  MP_TRY(nccl_check(ncclMemAlloc(&s.base, total), "ncclMemAlloc (tp symmetric)"));
  MP_TRY(nccl_check(ncclCommWindowRegister(c->tp_comm, s.base, total, &s.win, NCCL_WIN_COLL_SYMMETRIC),
                    "ncclCommWindowRegister"));
  ncclDevCommRequirements reqs{};
  reqs.lsaMultimem = true;
  auto* dev = new ncclDevComm{};
  ncclResult_t r = ncclDevCommCreate(c->tp_comm, &reqs, dev);
  if (r != ncclSuccess) {
    delete dev;
    tp_sym_free(c);
    s.tried = true;
    if (required) return nccl_check(r, "ncclDevCommCreate (multimem)");
    return MP_OK;
  }
  s.devcomm = dev;
  if (dev->lsaSize != c->t) {
    tp_sym_free(c);
    s.tried = true;
    if (required) return set_err(MP_EUNSUPPORTED, "TP group is not load/store accessible (lsa size %d)", dev->lsaSize);
    return MP_OK;
  }
  void** d_out = nullptr;
  MP_CUDA(cudaMalloc(&d_out, 2 * sizeof(void*)));
  tp_query_kernel<<<1, 1, 0, c->cs>>>(s.win, *dev, d_out);
  void* h_out[2] = {nullptr, nullptr};
  MP_CUDA(cudaMemcpyAsync(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost, c->cs));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  cudaFree(d_out);
  if (!h_out[0]) {
    tp_sym_free(c);
    s.tried = true;
    if (required) return set_err(MP_EUNSUPPORTED, "no multicast mapping for the TP window");
    return MP_OK;
  }
  s.mc = reinterpret_cast<char*>(h_out[0]);
  s.base = h_out[1];
  MP_CUDA(cudaMemsetAsync(s.base, 0, FLAG_BYTES, c->cs));
  // every rank's counter is zero before anyone arrives
  MP_TRY(nccl_check(ncclAllReduce(s.base, s.base, 1, ncclInt32, ncclSum, c->tp_comm, c->cs), "nvls setup barrier"));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  s.buf_bytes = buf_bytes;
  s.epoch = 0;
  s.next = 0;
  s.on = true;
  s.tried = true;
  return MP_OK;
}

// timing experiments only (results are wrong): MP_DEBUG_NVLS=local reads the
// local partial instead of the multicast sum, =nobarrier skips the barriers
static int debug_mode() {
  static const int m = [] {
    const char* e = getenv("MP_DEBUG_NVLS");
    if (!e) return 0;
    return std::string(e) == "local" ? 1 : std::string(e) == "nobarrier" ? 2 : 0;
  }();
  return m;
}

void tp_sym_next(mp_ctx* c, void** local, const void** mc) {
  TpSym& s = c->tps;
  const size_t off = FLAG_BYTES + (size_t)(s.next++ & 1) * s.buf_bytes;
  *local = reinterpret_cast<char*>(s.base) + off;
  *mc = s.mc + off;
}

bool tp_sym_two_shot(const mp_ctx* c) {
  static const int shot = getenv("MP_TP_NVLS_SHOT") ? atoi(getenv("MP_TP_NVLS_SHOT")) : 0;
  if (shot == 1) return false;
  if (shot == 2) return true;
  return c->t >= 4;
}

// slab [v0, v1) of 16-byte vectors: sum over the TP group (NVSwitch reduce-load,
// fp32 accumulation) multicast-stored to every rank's landing buffer
template <bool BF16>
__global__ void tp_rs_ag_kernel(const char* __restrict__ part_mc, char* __restrict__ land_mc, long long v0,
                                long long v1) {
  for (long long i = v0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < v1;
       i += (long long)gridDim.x * blockDim.x) {
    const char* src = part_mc + 16 * i;
    char* dst = land_mc + 16 * i;
    uint32_t a, b, cc, d;
    if constexpr (BF16) {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(cc), "=r"(d) : "l"(src) : "memory");
      asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(a), "r"(b),
                   "r"(cc), "r"(d) : "memory");
    } else {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a), "=r"(b), "=r"(cc), "=r"(d) : "l"(src) : "memory");
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(a), "r"(b),
                   "r"(cc), "r"(d) : "memory");
    }
  }
  __threadfence_system();   // stores performed before the following barrier's release
}

mp_status tp_sym_reduce_two_shot(mp_ctx* c, size_t n_elems, cudaStream_t st, const void** out) {
  TpSym& s = c->tps;
  const size_t slot = (size_t)((s.next - 1) & 1);
  const size_t poff = FLAG_BYTES + slot * s.buf_bytes, loff = FLAG_BYTES + (2 + slot) * s.buf_bytes;
  const long long nvec = (long long)(n_elems * c->esz / 16);
  const long long v0 = nvec * c->tp / c->t, v1 = nvec * (c->tp + 1) / c->t;
  MP_TRY(tp_sym_barrier(c, st));                      // all partial sums written
  const long long n = v1 - v0;
  const int grid = (int)std::max(1LL, std::min<long long>((n + 255) / 256, 4LL * num_sms()));
  if (c->cfg.dtype == MP_BF16)
    tp_rs_ag_kernel<true><<<grid, 256, 0, st>>>(s.mc + poff, s.mc + loff, v0, v1);
  else
    tp_rs_ag_kernel<false><<<grid, 256, 0, st>>>(s.mc + poff, s.mc + loff, v0, v1);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MP_ECUDA, "tp two-shot: %s", cudaGetErrorString(e));
  MP_TRY(tp_sym_barrier(c, st));                      // every slab stored on every rank
  *out = reinterpret_cast<char*>(s.base) + loff;
  return MP_OK;
}

bool tp_sym_debug_local() { return debug_mode() == 1; }

mp_status tp_sym_barrier(mp_ctx* c, cudaStream_t st) {
  TpSym& s = c->tps;
  if (debug_mode() == 2) return MP_OK;
  s.epoch++;
  tp_barrier_kernel<<<1, 32, 0, st>>>(reinterpret_cast<uint32_t*>(s.mc), reinterpret_cast<const uint32_t*>(s.base),
                                      s.epoch * (uint32_t)c->t);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(MP_ECUDA, "tp barrier: %s", cudaGetErrorString(e));
  return MP_OK;
}

}  // namespace mp
