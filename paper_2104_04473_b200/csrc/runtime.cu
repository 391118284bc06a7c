// Context, communicators, parameters and the pipeline stage runtime
// (mp_init / mp_set_weights / mp_layer_fwd / mp_layer_bwd / mp_run_batch).
//
// Pipeline runtime: each rank executes its
// static task order (schedule.h, identical to the oracle's) on one compute
// stream.  Stage boundaries are crossed over four directed FIFO channels per
// rank -- activations to the next device, activations from the previous one,
// gradients to the previous device, gradients from the next one -- each with
// its own stream (p2p.cu: CUDA-IPC receive rings in the peer's HBM, copy-engine
// copies over NVLink, slot flags written / awaited with stream memory
// operations, so no SM is held while a channel waits).  Every channel's send
// order equals its receiver's consume order (checked by the oracle for every
// schedule), so issuing receives in this rank's consume order cannot
// deadlock and keeps the ideal bubble.  A receive runs on the compute stream
// (wait for the slot's FULL flag, SM copy out of the slot, EMPTY flag), sends
// on their channel streams after the producing task's event.  After the flush the tied
// embedding gradient is all-reduced between the first and last stage and
// one Adam step updates every parameter (strict optimizer semantics).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "layer.h"
#include "runtime.h"

using namespace mp;

namespace {

inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

const char* kLayerNames[12] = {"ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                               "ln2_g", "ln2_b", "w_1",   "b_1",   "w_2", "b_2"};

std::string key(const std::string& n, int layer) { return n + "#" + std::to_string(layer); }

void add_param(mp_ctx* c, const std::string& name, int layer, int rows, int cols) {
  Param p;
  p.name = name; p.layer = layer; p.rows = rows; p.cols = cols;
  p.numel = (long long)rows * cols;
  p.off = c->n_params;
  c->n_params += (p.numel + 63) / 64 * 64;
  c->param_index[key(name, layer)] = (int)c->params.size();
  c->params.push_back(p);
}

bool is_layer_param(const std::string& n) {
  for (auto* s : kLayerNames)
    if (n == s) return true;
  return false;
}

// Map between the unpartitioned math-layout tensor (host) and this rank's
// storage shard.  For each storage element (r, c) returns the flat index in
// the unpartitioned tensor; also reports the math shape of the shard.
struct ShardMap {
  long long full_numel;
  int math_rows, math_cols;   // shard in math orientation
  bool transposed;            // storage = math^T
};

ShardMap shard_map(const mp_ctx* c, const std::string& n) {
  const int h = c->cfg.h, t = c->t;
  if (n == "w_qkv") return {3LL * h * h, h, 3 * h / t, true};
  if (n == "w_o") return {1LL * h * h, h / t, h, true};
  if (n == "w_1") return {4LL * h * h, h, 4 * h / t, true};
  if (n == "w_2") return {4LL * h * h, 4 * h / t, h, true};
  if (n == "b_qkv") return {3LL * h, 1, 3 * h / t, false};
  if (n == "b_1") return {4LL * h, 1, 4 * h / t, false};
  if (n == "emb") return {(long long)c->cfg.V * h, c->cfg.V / t, h, false};
  if (n == "pos") return {(long long)c->cfg.s * h, c->cfg.s, h, false};
  return {(long long)h, 1, h, false};
}

// index in the unpartitioned math tensor of math-shard element (i, j)
long long full_index(const mp_ctx* c, const std::string& n, int i, int j) {
  const int h = c->cfg.h, t = c->t, r = c->tp;
  if (n == "w_qkv") return (long long)i * 3 * h + (long long)r * 3 * h / t + j;
  if (n == "w_o") return ((long long)r * h / t + i) * h + j;
  if (n == "w_1") return (long long)i * 4 * h + (long long)r * 4 * h / t + j;
  if (n == "w_2") return ((long long)r * 4 * h / t + i) * h + j;
  if (n == "b_qkv") return (long long)r * 3 * h / t + j;
  if (n == "b_1") return (long long)r * 4 * h / t + j;
  if (n == "emb") return ((long long)r * (c->cfg.V / t) + i) * h + j;
  return (long long)i * shard_map(c, n).math_cols + j;
}

mp_status lookup(mp_ctx* c, const char* name, int layer, int* idx, bool* owned) {
  if (!name) return set_err(MP_EINVAL, "null name");
  std::string n(name);
  *owned = false;
  if (is_layer_param(n)) {
    if (layer < 0 || layer >= c->cfg.l) return set_err(MP_EINVAL, "layer %d out of range", layer);
    auto it = c->param_index.find(key(n, layer));
    if (it == c->param_index.end()) return MP_OK;
    *idx = it->second; *owned = true;
    return MP_OK;
  }
  if (n == "emb" || n == "pos" || n == "lnf_g" || n == "lnf_b") {
    auto it = c->param_index.find(key(n, -1));
    if (it == c->param_index.end()) return MP_OK;
    *idx = it->second; *owned = true;
    return MP_OK;
  }
  return set_err(MP_EINVAL, "unknown parameter name '%s'", name);
}

mp_status cast_store(mp_ctx* c, long long off, long long n, cudaStream_t st) {
  if (c->cfg.dtype == MP_BF16)
    return cast_from_f32<__nv_bfloat16>(c->master + off, reinterpret_cast<__nv_bfloat16*>(c->wstore) + off, n, st);
  return MP_OK;  // fp32: storage aliases the master copy
}

struct EvPool {
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  unsigned flags = cudaEventDisableTiming;
  cudaEvent_t get() {
    if (next == ev.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, flags);
      ev.push_back(e);
    }
    return ev[next++];
  }
  void destroy() {
    for (auto e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};

struct RuntimeExtra {
  EvPool sync, timing;
};
std::map<const mp_ctx*, RuntimeExtra> g_extra;

}  // namespace

extern "C" {

int mp_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

mp_status mp_nccl_get_id(void* out) {
  if (!out) return set_err(MP_EINVAL, "null out");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(MP_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out, &id, sizeof(id));
  return MP_OK;
}

mp_status mp_init(int t, int p, int v, int d, const mp_model_cfg* cfg, int world_rank, int world_size,
                  int local_device, const void* nccl_id, mp_ctx** out) {
  if (!out || !cfg || !nccl_id) return set_err(MP_EINVAL, "null argument");
  *out = nullptr;
  MP_TRY(validate_cfg(cfg, t, p, v, d));
  if (t * p * d != world_size) return set_err(MP_EDIV, "t*p*d=%d != world size %d", t * p * d, world_size);
  if (world_rank < 0 || world_rank >= world_size) return set_err(MP_EINVAL, "bad rank");
  if (cfg->p_drop_attn < 0.f || cfg->p_drop_attn >= 1.f || cfg->p_drop_hidden < 0.f || cfg->p_drop_hidden >= 1.f)
    return set_err(MP_EINVAL, "dropout rates must be in [0, 1)");
  if (cfg->dtype != MP_BF16 && cfg->dtype != MP_FP32) return set_err(MP_EINVAL, "bad dtype");
  if (p > 1) {
    // Six library streams (+ the caller's): with fewer hardware queues a channel
    // stream's cuStreamWaitValue32 on a peer's flag can sit in a queue shared
    // with another stream's work and block it (a false dependency that can
    // deadlock the pipeline).
    const char* mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    if (mc && atoi(mc) < 8)
      return set_err(MP_EINVAL, "CUDA_DEVICE_MAX_CONNECTIONS=%s is too small for p > 1 (need >= 8, use 32)", mc);
  }
  MP_CUDA(cudaSetDevice(local_device));
  MP_REQUIRE_DEVICE();
  mp_ctx* c = new mp_ctx();
  c->t = t; c->p = p; c->v = v; c->d = d; c->rank = world_rank; c->world = world_size; c->device = local_device;
  c->tp = world_rank % t;
  c->pp = (world_rank / t) % p;
  c->dp = world_rank / (t * p);
  c->cfg = *cfg;
  if (c->cfg.ln_eps <= 0.f) c->cfg.ln_eps = 1e-5f;
  c->esz = cfg->dtype == MP_BF16 ? 2 : 4;
  c->nccl_dt = cfg->dtype == MP_BF16 ? ncclBfloat16 : ncclFloat32;
  // ---- streams, pool, events
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  MP_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  MP_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  MP_CUDA(cudaStreamCreateWithPriority(&c->s_act_send, cudaStreamNonBlocking, hi));
  MP_CUDA(cudaStreamCreateWithPriority(&c->s_act_recv, cudaStreamNonBlocking, hi));
  MP_CUDA(cudaStreamCreateWithPriority(&c->s_grad_send, cudaStreamNonBlocking, hi));
  MP_CUDA(cudaStreamCreateWithPriority(&c->s_grad_recv, cudaStreamNonBlocking, hi));
  MP_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, local_device));
  uint64_t thr = UINT64_MAX;
  MP_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
  {
    // Buffers freed on a pipeline-channel stream (which can block on a peer's flag) must never
    // make the compute stream wait on that stream through a pool-inserted dependency: that
    // would couple this rank's compute to the peer's progress (a possible cross-rank cycle).
    // Event-ordered reuse stays on; internal dependencies are off.
    int zero = 0;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
  }
  if (getenv("MP_POOL_NOREUSE")) {
    int zero = 0;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseFollowEventDependencies, &zero);
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowOpportunistic, &zero);
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
  }
  for (int i = 0; i < 2; ++i) {
    cudaEvent_t e;
    MP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->events.push_back(e);
  }
  g_extra[c].timing.flags = cudaEventDefault;
  // ---- communicators (P:185-189 grid; rank = (dp p + pp) t + tp)
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&c->world_comm, world_size, id, world_rank);
  if (r != ncclSuccess) { delete c; return set_err(MP_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)); }
  if (t > 1) {
    r = ncclCommSplit(c->world_comm, c->dp * p + c->pp, c->tp, &c->tp_comm, nullptr);
    if (r != ncclSuccess) return set_err(MP_ENCCL, "tp split: %s", ncclGetErrorString(r));
  }
  if (p > 1) {
    // tied word embedding: stage 0 and stage S-1 hold copies of E_r (pipeline
    // activations / gradients travel over the IPC channels of p2p.cu)
    const bool tie = c->pp == 0 || c->pp == p - 1;
    r = ncclCommSplit(c->world_comm, tie ? c->dp * t + c->tp : NCCL_SPLIT_NOCOLOR, c->pp == 0 ? 0 : 1, &c->emb_comm,
                      nullptr);
    if (r != ncclSuccess) return set_err(MP_ENCCL, "embedding split: %s", ncclGetErrorString(r));
  }
  if (d > 1) {
    // data parallelism: replicas of the same (pp, tp) shard sum their gradients
    r = ncclCommSplit(c->world_comm, c->pp * t + c->tp, c->dp, &c->dp_comm, nullptr);
    if (r != ncclSuccess) return set_err(MP_ENCCL, "dp split: %s", ncclGetErrorString(r));
    MP_CUDA(cudaStreamCreateWithPriority(&c->s_dp, cudaStreamNonBlocking, lo));
  }
  // ---- stage map and parameters
  c->dev_of_layer.resize(cfg->l);
  c->chunk_of_layer.resize(cfg->l);
  mp_get_stage_map(cfg->l, p, v, c->dev_of_layer.data(), c->chunk_of_layer.data());
  c->has_emb = c->pp == 0;
  c->has_head = c->pp == p - 1;
  const int h = cfg->h;
  for (int k = 0; k < cfg->l; ++k) {
    if (c->dev_of_layer[k] != c->pp) continue;
    LayerParams lp;
    const int shapes[12][2] = {{1, h}, {1, h}, {3 * h / t, h}, {1, 3 * h / t}, {h, h / t}, {1, h},
                               {1, h}, {1, h}, {4 * h / t, h}, {1, 4 * h / t}, {h, 4 * h / t}, {1, h}};
    for (int i = 0; i < 12; ++i) {
      lp.idx[i] = (int)c->params.size();
      add_param(c, kLayerNames[i], k, shapes[i][0], shapes[i][1]);
    }
    c->layer_params[k] = lp;
  }
  if (c->has_emb || c->has_head) add_param(c, "emb", -1, cfg->V / t, h);
  if (c->has_emb) add_param(c, "pos", -1, cfg->s, h);
  if (c->has_head) { add_param(c, "lnf_g", -1, 1, h); add_param(c, "lnf_b", -1, 1, h); }
  const size_t nb = (size_t)c->n_params;
  MP_CUDA(cudaMalloc(&c->master, nb * 4));
  MP_CUDA(cudaMemset(c->master, 0, nb * 4));
  if (cfg->dtype == MP_BF16) {
    MP_CUDA(cudaMalloc(&c->wstore, nb * 2));
    MP_CUDA(cudaMemset(c->wstore, 0, nb * 2));
  } else {
    c->wstore = c->master;
  }
  MP_CUDA(cudaMalloc(&c->grads, nb * 4));
  MP_CUDA(cudaMemset(c->grads, 0, nb * 4));
  MP_CUDA(cudaMalloc(&c->d_loss, 256));
  MP_CUDA(cudaDeviceSynchronize());
  *out = c;
  return MP_OK;
}

mp_status mp_finalize(mp_ctx* c) {
  if (!c) return MP_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->slots) stash_release(c, kv.second, c->cs);
  cudaStreamSynchronize(c->cs);
  p2p_release(c);
  tp_sym_free(c);
  ncclComm_t comms[] = {c->tp_comm, c->emb_comm, c->dp_comm, c->world_comm};
  for (auto cm : comms)
    if (cm) ncclCommDestroy(cm);
  void* bufs[] = {c->ws_z, c->ws_dsq, c->ws_d4h, c->ws_dh1, c->ws_dh2, c->ws_dqkv, c->ws_dctx, c->ws_fa,
                  c->grads, c->adam_m, c->adam_v, c->d_loss, c->master, c->head_dl, c->head_z};
  for (void* q : bufs)
    if (q) cudaFree(q);
  if (c->cfg.dtype == MP_BF16 && c->wstore) cudaFree(c->wstore);
  for (auto e : c->events) cudaEventDestroy(e);
  auto it = g_extra.find(c);
  if (it != g_extra.end()) { it->second.sync.destroy(); it->second.timing.destroy(); g_extra.erase(it); }
  cudaStream_t ss[] = {c->cs, c->side, c->s_act_send, c->s_act_recv, c->s_grad_send, c->s_grad_recv, c->s_dp};
  for (auto s : ss)
    if (s) cudaStreamDestroy(s);
  delete c;
  return MP_OK;
}

}  // extern "C"

template <class H>
static mp_status set_weights_t(mp_ctx* c, const char* name, int layer, const H* host) {
  if (!c || !host) return set_err(MP_EINVAL, "null argument");
  int idx = -1; bool owned = false;
  MP_TRY(lookup(c, name, layer, &idx, &owned));
  if (!owned) return MP_OK;
  MP_CUDA(cudaSetDevice(c->device));
  const Param& P = c->params[idx];
  const ShardMap sm = shard_map(c, P.name);
  std::vector<float> st((size_t)P.numel);
  for (int i = 0; i < sm.math_rows; ++i)
    for (int j = 0; j < sm.math_cols; ++j) {
      const float val = (float)host[full_index(c, P.name, i, j)];   // fp64 input: rounded once
      if (sm.transposed) st[(size_t)j * sm.math_rows + i] = val;
      else st[(size_t)i * sm.math_cols + j] = val;
    }
  // same stream as the cast: a pageable cudaMemcpy may return before its DMA lands
  MP_CUDA(cudaMemcpyAsync(c->master + P.off, st.data(), st.size() * 4, cudaMemcpyHostToDevice, c->cs));
  MP_TRY(cast_store(c, P.off, P.numel, c->cs));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  return MP_OK;
}

extern "C" {

mp_status mp_set_weights(mp_ctx* c, const char* name, int layer, const float* host) {
  return set_weights_t(c, name, layer, host);
}
mp_status mp_set_weights_f64(mp_ctx* c, const char* name, int layer, const double* host) {
  return set_weights_t(c, name, layer, host);
}

static mp_status get_common(mp_ctx* c, const char* name, int layer, float* host, long long* n, const float* base) {
  if (!c || !n) return set_err(MP_EINVAL, "null argument");
  int idx = -1; bool owned = false;
  MP_TRY(lookup(c, name, layer, &idx, &owned));
  if (!owned) return set_err(MP_EINVAL, "parameter %s of layer %d is not on this rank", name, layer);
  const Param& P = c->params[idx];
  *n = P.numel;
  if (!host) return MP_OK;
  MP_CUDA(cudaSetDevice(c->device));
  MP_CUDA(cudaDeviceSynchronize());
  const ShardMap sm = shard_map(c, P.name);
  std::vector<float> st((size_t)P.numel);
  MP_CUDA(cudaMemcpy(st.data(), base + P.off, st.size() * 4, cudaMemcpyDeviceToHost));
  for (int i = 0; i < sm.math_rows; ++i)
    for (int j = 0; j < sm.math_cols; ++j)
      host[(size_t)i * sm.math_cols + j] = sm.transposed ? st[(size_t)j * sm.math_rows + i] : st[(size_t)i * sm.math_cols + j];
  return MP_OK;
}

mp_status mp_get_weights(mp_ctx* c, const char* name, int layer, float* host, long long* n) {
  return get_common(c, name, layer, host, n, c ? c->master : nullptr);
}
mp_status mp_get_grads(mp_ctx* c, const char* name, int layer, float* host, long long* n) {
  return get_common(c, name, layer, host, n, c ? c->grads : nullptr);
}

mp_status mp_zero_grads(mp_ctx* c) {
  if (!c) return set_err(MP_EINVAL, "null ctx");
  MP_CUDA(cudaSetDevice(c->device));
  MP_CUDA(cudaMemsetAsync(c->grads, 0, (size_t)c->n_params * 4, c->cs));
  MP_CUDA(cudaStreamSynchronize(c->cs));
  return MP_OK;
}

// ------------------------------------------------------------ layer calls
mp_status mp_layer_fwd(mp_ctx* c, int layer, int b, const void* x, void* y, int* stash_slot, void* stream) {
  if (!c || !x || !y || !stash_slot) return set_err(MP_EINVAL, "null argument");
  if (layer < 0 || layer >= c->cfg.l || !c->layer_params.count(layer))
    return set_err(MP_EINVAL, "layer %d is not on this rank", layer);
  if (b < 1) return set_err(MP_EINVAL, "b must be >= 1");
  MP_CUDA(cudaSetDevice(c->device));
  cudaStream_t saved = c->cs;
  c->cs = reinterpret_cast<cudaStream_t>(stream);   // NULL = legacy default stream (header contract)
  LayerStash st;
  c->cur_seq0 = 0;
  const size_t bytes = (size_t)c->cfg.s * b * c->cfg.h * c->esz;
  mp_status s = alloc_async(c, &st.x, bytes, c->cs);
  if (s == MP_OK) {
    cudaMemcpyAsync(st.x, x, bytes, cudaMemcpyDeviceToDevice, c->cs);
    st.own_x = true;
    s = layer_fwd(c, layer, b, st.x, y, st);
  }
  c->cs = saved;
  if (s != MP_OK) return s;
  const int id = c->next_slot++;
  c->slots[id] = st;
  *stash_slot = id;
  return MP_OK;
}

mp_status mp_layer_bwd(mp_ctx* c, int layer, int b, int slot, const void* dy, void* dx, void* stream) {
  if (!c || !dy || !dx) return set_err(MP_EINVAL, "null argument");
  auto it = c->slots.find(slot);
  if (it == c->slots.end()) return set_err(MP_ESTATE, "unknown stash slot %d", slot);
  if (!c->layer_params.count(layer)) return set_err(MP_EINVAL, "layer %d is not on this rank", layer);
  if (it->second.b != b) return set_err(MP_EINVAL, "b differs from the forward");
  MP_CUDA(cudaSetDevice(c->device));
  cudaStream_t saved = c->cs;
  c->cs = reinterpret_cast<cudaStream_t>(stream);   // NULL = legacy default stream
  mp_status s = layer_bwd(c, layer, it->second, dy, dx);
  if (s == MP_OK) s = stash_release(c, it->second, c->cs);
  c->cs = saved;
  c->slots.erase(it);
  return s;
}

mp_status mp_head_fwd_bwd(mp_ctx* c, int b, const void* x, const int* labels, int labels_ld, float scale, void* dx,
                          float* loss_dev, void* stream) {
  if (!c || !x || !labels || !dx || !loss_dev) return set_err(MP_EINVAL, "null argument");
  if (!c->has_head) return set_err(MP_EINVAL, "rank %d (pp=%d) holds no head: only the last stage does", c->rank, c->pp);
  if (b < 1 || labels_ld < c->cfg.s) return set_err(MP_EINVAL, "need b >= 1 and labels_ld >= s");
  MP_CUDA(cudaSetDevice(c->device));
  cudaStream_t saved = c->cs;
  c->cs = reinterpret_cast<cudaStream_t>(stream);   // NULL = legacy default stream
  mp_status s = MP_OK;
  if (cudaMemsetAsync(c->d_loss, 0, 4, c->cs) != cudaSuccess) s = set_err(MP_ECUDA, "memset");
  if (s == MP_OK) s = head_fwd_bwd(c, x, labels, labels_ld, b, scale, dx);
  if (s == MP_OK && cudaMemcpyAsync(loss_dev, c->d_loss, 4, cudaMemcpyDeviceToDevice, c->cs) != cudaSuccess)
    s = set_err(MP_ECUDA, "loss copy");
  c->cs = saved;
  return s;
}

// ------------------------------------------------------------- batch call
static mp_status run_batch_impl(mp_ctx* c, int B, int b, int m, mp_schedule sched, const int* tokens, bool tok_dev,
                                int apply_optimizer, float* loss_host, float* loss_dev, mp_batch_stats* stats) {
  if (!c || !tokens || (!loss_host && !loss_dev)) return set_err(MP_EINVAL, "null argument");
  if (b < 1 || m < 1 || B != m * b * c->d) return set_err(MP_EDIV, "need B = m b d (P:189): B=%d b=%d m=%d", B, b, m);
  if ((sched == MP_GPIPE || sched == MP_1F1B) && c->v != 1)
    return set_err(MP_ESCHED, "context built with v=%d needs the interleaved schedule", c->v);
  std::vector<Task> tasks;
  MP_TRY(build_schedule(c->p, m, c->v, sched, c->pp, tasks));
  MP_CUDA(cudaSetDevice(c->device));
  MP_TRY(ensure_workspace(c, b));
  RuntimeExtra& X = g_extra[c];
  X.sync.next = 0;
  X.timing.next = 0;
  const int s = c->cfg.s, h = c->cfg.h, p = c->p, v = c->v, S = p * v;
  const int Lc = c->cfg.l / S;
  const size_t act_elems = (size_t)s * b * h, act_bytes = act_elems * c->esz;
  const float scale = 1.f / ((float)B * (float)s);
  cudaStream_t cs = c->cs;
  const bool recompute = c->cfg.recompute != 0;

  MP_TRY(p2p_ensure(c, act_bytes));
  cudaEvent_t ev_start = X.timing.get(), ev_end = X.timing.get();
  MP_CUDA(cudaEventRecord(ev_start, cs));
  // tokens -> device (inputs x = tok[:, :s], labels y = tok[:, 1:])
  // this data-parallel replica's rows [dp B/d, (dp+1) B/d) of the batch
  const size_t rows = (size_t)m * b;
  const int* tok_mine = tokens + (size_t)c->dp * rows * (s + 1);
  int* dtok = nullptr;
  if (tok_dev) {
    dtok = const_cast<int*>(tok_mine);
  } else {
    MP_TRY(alloc_async(c, (void**)&dtok, sizeof(int) * rows * (s + 1), cs));
    MP_CUDA(cudaMemcpyAsync(dtok, tok_mine, sizeof(int) * rows * (s + 1), cudaMemcpyHostToDevice, cs));
  }
  MP_CUDA(cudaMemsetAsync(c->grads, 0, (size_t)c->n_params * 4, cs));
  MP_CUDA(cudaMemsetAsync(c->d_loss, 0, 4, cs));

  std::map<std::pair<int, int>, LayerStash> stash;        // (mb, layer)
  std::map<std::pair<int, int>, void*> local_act, local_grad;   // (mb, stage) hand-offs on this device
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> task_ev;
  int inflight = 0, peak = 0;
  mp_status st = MP_OK;
  // data parallelism: once a layer's last backward (its m-th) is enqueued, its gradient
  // segment is all-reduced over the replicas on s_dp while the remaining layers' backward
  // runs.  Only at t = 1: with t > 1 the TP reductions are spinning kernels / NCCL kernels
  // of another communicator whose relative order across ranks would not be fixed.
  const bool dp_overlap = c->dp_comm && c->t == 1 && !getenv("MP_DP_NO_OVERLAP");
  std::map<int, int> bwd_count;
  long long model_off = c->n_params;   // first model-level (emb / pos / lnf) element; layers precede it
  for (const auto& P : c->params)
    if (P.layer < 0) model_off = std::min(model_off, P.off);

  // logit-layer weight gradient deferred to the flush (bf16 last stage): per microbatch
  // dlogits [T, V/t] and Z [T, h] are kept (MP_HEAD_DEFER_GB bounds the buffers, default 16)
  bool defer_dE = false;
  if (c->has_head && c->cfg.dtype == MP_BF16 && !getenv("MP_HEAD_FP32_LOGITS")) {
    static const double budget = getenv("MP_HEAD_DEFER_GB") ? atof(getenv("MP_HEAD_DEFER_GB")) : 16.0;
    const size_t dl = (size_t)m * s * b * (size_t)(c->cfg.V / c->t) * 2, zb = (size_t)m * s * b * h * 2;
    if ((double)(dl + zb) <= budget * 1e9) {
      defer_dE = true;
      if (c->head_dl_bytes < dl || c->head_z_bytes < zb) {
        MP_CUDA(cudaStreamSynchronize(cs));
        if (c->head_dl) cudaFree(c->head_dl);
        if (c->head_z) cudaFree(c->head_z);
        c->head_dl = c->head_z = nullptr;
        c->head_dl_bytes = c->head_z_bytes = 0;
        MP_CUDA(cudaMalloc(&c->head_dl, dl));
        MP_CUDA(cudaMalloc(&c->head_z, zb));
        c->head_dl_bytes = dl;
        c->head_z_bytes = zb;
      }
    }
  }
  static const bool dbg = getenv("MP_DEBUG") != nullptr;
  for (const Task& tk : tasks) {
    const int sigma = tk.chunk * p + c->pp;
    if (dbg) fprintf(stderr, "[mp rank %d] enqueue %c mb=%d chunk=%d stage=%d\n", c->rank, tk.kind ? 'B' : 'F', tk.mb,
                     tk.chunk, sigma);
    const int* tok = dtok + (size_t)tk.mb * b * (s + 1);
    c->cur_seq0 = (c->dp * m + tk.mb) * b;   // global index of the microbatch's first sequence (dropout counters)
    if (tk.kind == 0) {
      // ------------------------------------------------------------ forward
      void* x = nullptr;
      if (sigma == 0) {
        MP_TRY(alloc_async(c, &x, act_bytes, cs));
      } else if (p == 1) {
        x = local_act.at({tk.mb, sigma});
        local_act.erase({tk.mb, sigma});
      } else {
        // received on the compute stream itself: it waits for the slot's FULL flag, copies the
        // slot with an SM kernel and frees it (no channel-stream / event hop on the critical path)
        MP_TRY(alloc_async(c, &x, act_bytes, cs));
        MP_TRY(p2p_recv_act(c, x, act_bytes, cs));
      }
      cudaEvent_t t0 = X.timing.get(), t1 = X.timing.get();
      MP_CUDA(cudaEventRecord(t0, cs));
      if (sigma == 0) MP_TRY(embed_forward(c, tok, s + 1, b, x));
      for (int k = sigma * Lc; k < (sigma + 1) * Lc; ++k) {
        void* y = nullptr;
        MP_TRY(alloc_async(c, &y, act_bytes, cs));
        LayerStash ls;
        ls.x = x; ls.own_x = true;
        MP_TRY(layer_fwd(c, k, b, x, y, ls));
        if (recompute) {    // activation recomputation: keep only the layer input
          MP_CUDA(cudaFreeAsync(ls.block, cs));
          ls.block = nullptr;
        }
        stash[{tk.mb, k}] = ls;
        x = y;
      }
      ++inflight;
      peak = std::max(peak, inflight);
      if (sigma == S - 1) {
        void* dx = nullptr;
        MP_TRY(alloc_async(c, &dx, act_bytes, cs));
        MP_TRY(head_fwd_bwd(c, x, tok + 1, s + 1, b, scale, dx, defer_dE ? tk.mb : -1));
        MP_CUDA(cudaFreeAsync(x, cs));
        local_grad[{tk.mb, sigma}] = dx;
        MP_CUDA(cudaEventRecord(t1, cs));
      } else if (p == 1) {
        local_act[{tk.mb, sigma + 1}] = x;
        MP_CUDA(cudaEventRecord(t1, cs));
      } else {
        MP_CUDA(cudaEventRecord(t1, cs));
        MP_CUDA(cudaStreamWaitEvent(c->s_act_send, t1, 0));
        MP_TRY(p2p_send_act(c, x, act_bytes, c->s_act_send));
        MP_CUDA(cudaFreeAsync(x, c->s_act_send));
      }
      task_ev.push_back({t0, t1});
      if (dbg && getenv("MP_DEBUG")[0] == '2') {
        cudaError_t e2 = cudaStreamSynchronize(cs);
        fprintf(stderr, "[mp rank %d] done F mb=%d (%s)\n", c->rank, tk.mb, cudaGetErrorString(e2));
      }
    } else {
      // ----------------------------------------------------------- backward
      void* dy = nullptr;
      if (sigma == S - 1 || p == 1) {
        dy = local_grad.at({tk.mb, sigma});
        local_grad.erase({tk.mb, sigma});
      } else {
        MP_TRY(alloc_async(c, &dy, act_bytes, cs));
        MP_TRY(p2p_recv_grad(c, dy, act_bytes, cs));
      }
      cudaEvent_t t0 = X.timing.get(), t1 = X.timing.get();
      MP_CUDA(cudaEventRecord(t0, cs));
      for (int k = (sigma + 1) * Lc - 1; k >= sigma * Lc; --k) {
        void* dx = nullptr;
        MP_TRY(alloc_async(c, &dx, act_bytes, cs));
        LayerStash& ls = stash.at({tk.mb, k});
        if (recompute) {    // re-run the layer forward from its checkpointed input (one extra forward)
          void* y = nullptr;
          MP_TRY(alloc_async(c, &y, act_bytes, cs));
          MP_TRY(layer_fwd(c, k, b, ls.x, y, ls));
          MP_CUDA(cudaFreeAsync(y, cs));
        }
        MP_TRY(layer_bwd(c, k, ls, dy, dx));
        if (dp_overlap && ++bwd_count[k] == m) {
          const auto& ix = c->layer_params.at(k).idx;
          const long long lo = c->params[ix[0]].off, hi = c->params[ix[11]].off + c->params[ix[11]].numel;
          cudaEvent_t e = X.sync.get();
          MP_CUDA(cudaEventRecord(e, cs));
          MP_CUDA(cudaStreamWaitEvent(c->s_dp, e, 0));
          MP_TRY(nccl_check(ncclAllReduce(c->grads + lo, c->grads + lo, (size_t)(hi - lo), ncclFloat32, ncclSum,
                                          c->dp_comm, c->s_dp), "data-parallel layer gradient all-reduce"));
        }
        MP_TRY(stash_release(c, ls, cs));
        stash.erase({tk.mb, k});
        MP_CUDA(cudaFreeAsync(dy, cs));
        dy = dx;
      }
      --inflight;
      if (sigma == 0) {
        MP_TRY(embed_backward(c, tok, s + 1, b, dy));
        MP_CUDA(cudaFreeAsync(dy, cs));
        MP_CUDA(cudaEventRecord(t1, cs));
      } else if (p == 1) {
        local_grad[{tk.mb, sigma - 1}] = dy;
        MP_CUDA(cudaEventRecord(t1, cs));
      } else {
        MP_CUDA(cudaEventRecord(t1, cs));
        MP_CUDA(cudaStreamWaitEvent(c->s_grad_send, t1, 0));
        MP_TRY(p2p_send_grad(c, dy, act_bytes, c->s_grad_send));
        MP_CUDA(cudaFreeAsync(dy, c->s_grad_send));
      }
      task_ev.push_back({t0, t1});
      if (dbg && getenv("MP_DEBUG")[0] == '2') {
        cudaError_t e2 = cudaStreamSynchronize(cs);
        fprintf(stderr, "[mp rank %d] done B mb=%d (%s)\n", c->rank, tk.mb, cudaGetErrorString(e2));
      }
    }
  }
  // ------------------------------------------------------------------ flush
  if (dbg) fprintf(stderr, "[mp rank %d] all tasks enqueued\n", c->rank);
  if (defer_dE) MP_TRY(head_dE_deferred(c, b, m));
  if (p > 1) {
    cudaStream_t ss[] = {c->s_act_send, c->s_grad_send, c->s_act_recv, c->s_grad_recv};
    for (auto q : ss) {
      cudaEvent_t e = X.sync.get();
      MP_CUDA(cudaEventRecord(e, q));
      MP_CUDA(cudaStreamWaitEvent(cs, e, 0));
    }
    // tied word embedding: stage 0 and stage S-1 hold copies of E_r; sum their gradients
    if (c->emb_comm && (c->has_emb || c->has_head)) {
      const Param& P = c->params[c->param_index.at("emb#-1")];
      MP_TRY(nccl_check(ncclAllReduce(c->grads + P.off, c->grads + P.off, P.numel, ncclFloat32, ncclSum, c->emb_comm, cs),
                        "embedding grad all-reduce"));
    }
  }
  // data parallelism: sum the replicas' gradients (each already carries the 1/(B s) global-batch scale)
  if (c->dp_comm) {
    long long lo = 0;
    if (dp_overlap) {   // the layers' segments are already in flight on s_dp
      cudaEvent_t e = X.sync.get();
      MP_CUDA(cudaEventRecord(e, c->s_dp));
      MP_CUDA(cudaStreamWaitEvent(cs, e, 0));
      lo = model_off;
    }
    if (c->n_params > lo)
      MP_TRY(nccl_check(ncclAllReduce(c->grads + lo, c->grads + lo, (size_t)(c->n_params - lo), ncclFloat32, ncclSum,
                                      c->dp_comm, cs), "data-parallel gradient all-reduce"));
  }
  // loss: contributed by (last stage, tp 0) of every replica, then shared with every rank
  {
    const bool contrib = c->has_head && c->tp == 0;
    float* red = c->d_loss + 32;
    if (contrib) MP_CUDA(cudaMemcpyAsync(red, c->d_loss, 4, cudaMemcpyDeviceToDevice, cs));
    else MP_CUDA(cudaMemsetAsync(red, 0, 4, cs));
    if (c->world > 1)
      MP_TRY(nccl_check(ncclAllReduce(red, red, 1, ncclFloat32, ncclSum, c->world_comm, cs), "loss all-reduce"));
  }
  if (apply_optimizer) {
    const size_t nb = (size_t)c->n_params * 4;
    if (!c->adam_m) {
      MP_CUDA(cudaMalloc(&c->adam_m, nb));
      MP_CUDA(cudaMalloc(&c->adam_v, nb));
      MP_CUDA(cudaMemsetAsync(c->adam_m, 0, nb, cs));
      MP_CUDA(cudaMemsetAsync(c->adam_v, 0, nb, cs));
    }
    c->adam_step++;
    const float b1 = 0.9f, b2 = 0.999f;
    const float bc1 = 1.f - std::pow(b1, (float)c->adam_step), bc2 = 1.f - std::pow(b2, (float)c->adam_step);
    if (c->cfg.dtype == MP_BF16)
      MP_TRY(adam_step<__nv_bfloat16>(c->master, c->grads, c->adam_m, c->adam_v,
                                      reinterpret_cast<__nv_bfloat16*>(c->wstore), c->n_params, c->cfg.lr, b1, b2,
                                      1e-8f, bc1, bc2, cs));
    else
      MP_TRY(adam_step<float>(c->master, c->grads, c->adam_m, c->adam_v, c->master, c->n_params, c->cfg.lr, b1, b2,
                              1e-8f, bc1, bc2, cs));
  }
  if (!tok_dev) MP_CUDA(cudaFreeAsync(dtok, cs));
  if (loss_host) {
    MP_CUDA(cudaMemcpyAsync(loss_host, c->d_loss + 32, 4, cudaMemcpyDeviceToHost, cs));
  } else {
    MP_CUDA(cudaMemcpyAsync(loss_dev, c->d_loss + 32, 4, cudaMemcpyDeviceToDevice, cs));
  }
  MP_CUDA(cudaEventRecord(ev_end, cs));
  if (loss_host || stats) MP_CUDA(cudaStreamSynchronize(cs));
  if (!stash.empty() || !local_act.empty() || !local_grad.empty())
    return set_err(MP_ESTATE, "pipeline finished with live activations (schedule bug)");
  if (stats) {
    float ms = 0.f, pipe_ms = 0.f;
    cudaEventElapsedTime(&ms, ev_start, ev_end);
    if (!task_ev.empty()) cudaEventElapsedTime(&pipe_ms, ev_start, task_ev.back().second);
    double busy = 0.0, tf = 0.0, tb = 0.0;
    int nf = 0, nb = 0;
    for (size_t i = 0; i < task_ev.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, task_ev[i].first, task_ev[i].second);
      busy += t;
      if (tasks[i].kind == 0) { tf += t; ++nf; } else { tb += t; ++nb; }
    }
    stats->iter_seconds = ms * 1e-3;
    stats->busy_seconds = busy * 1e-3;
    stats->pipeline_seconds = pipe_ms * 1e-3;
    stats->t_fwd_task = nf ? tf * 1e-3 / nf : 0.0;
    stats->t_bwd_task = nb ? tb * 1e-3 / nb : 0.0;
    stats->model_flops = mp_flops(B, s, c->cfg.l, h, c->cfg.V, c->cfg.recompute);
    stats->model_tflops_per_gpu = stats->model_flops / (c->world * stats->iter_seconds) / 1e12;
    // idle share of this rank between the batch start and its last task (the flush, the
    // tied-embedding all-reduce and the optimizer step are not part of the bubble)
    stats->bubble_measured = busy > 0 ? (pipe_ms - busy) / busy : 0.0;
    stats->bubble_formula = (double)(p - 1) / (sched == MP_INTERLEAVED ? (double)v * m : (double)m);
    stats->peak_inflight = peak;
    stats->n_tasks = (int)tasks.size();
  }
  (void)st;
  return MP_OK;
}

mp_status mp_run_batch(mp_ctx* c, int B, int b, int m, mp_schedule sched, const int* tokens, int apply_optimizer,
                       float* loss_out, mp_batch_stats* stats) {
  return run_batch_impl(c, B, b, m, sched, tokens, false, apply_optimizer, loss_out, nullptr, stats);
}

int mp_tp_comm_mode(const mp_ctx* c) {
  if (!c) return MP_TP_COMM_AUTO;
  if (c->t == 1) return MP_TP_COMM_NCCL;
  if (!c->tps.tried) return MP_TP_COMM_AUTO;
  return c->tps.on ? MP_TP_COMM_NVLS : MP_TP_COMM_NCCL;
}

mp_status mp_tp_reduce_probe(mp_ctx* c, int b, int iters, double* seconds) {
  if (!c || !seconds || b < 1 || iters < 1) return set_err(MP_EINVAL, "bad argument");
  if (c->t == 1) return set_err(MP_EUNSUPPORTED, "tp probe: t = 1 has no tensor-parallel reduction");
  MP_CUDA(cudaSetDevice(c->device));
  return tp_reduce_probe(c, b, iters, seconds);
}

void* mp_compute_stream(mp_ctx* c) { return c ? reinterpret_cast<void*>(c->cs) : nullptr; }

mp_status mp_run_batch_dev(mp_ctx* c, int B, int b, int m, mp_schedule sched, const int* d_tokens,
                           int apply_optimizer, float* d_loss, mp_batch_stats* stats) {
  return run_batch_impl(c, B, b, m, sched, d_tokens, true, apply_optimizer, nullptr, d_loss, stats);
}

}  // extern "C"
