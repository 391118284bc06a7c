// Per-process runtime state of the PTD-P hot path: process grid, NCCL
// communicators, weight shards, gradient accumulators, Adam state,
// activation stash and workspaces.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/mp.h"
#include "p2p.h"
#include "schedule.h"
#include "tpcomm.h"

namespace mp {

// One parameter tensor of this rank, inside the flat parameter arrays.
// Weight matrices are stored transposed w.r.t. the math orientation
// (row = output feature, contiguous = input feature: "K-major" for the
// forward GEMM), e.g. W_qkv shard [3h/t, h].
struct Param {
  std::string name;
  int layer;           // -1 for model-level parameters
  long long off;       // element offset in the flat arrays
  long long numel;
  int rows, cols;      // storage shape
};

struct LayerParams {
  int idx[12];         // indices into ctx->params for ln1_g .. b_2
};

// Activations stashed by one layer forward for its backward.
struct LayerStash {
  void* x = nullptr;   // layer input [T, h]
  bool own_x = false;  // freed with the stash
  void* block = nullptr;  // single allocation holding everything below
  float *mu1, *rs1, *mu2, *rs2;
  void *A, *QKV, *P, *ctx, *X1, *A2, *Y1, *H;
  int b = 1;
  int seq0 = 0;        // global index of the microbatch's first sequence (dropout counters)
};

struct HeadStash {
  void* block = nullptr;
};

}  // namespace mp

struct mp_ctx {
  // process grid, rank = (dp * p + pp) * t + tp
  int t, p, v, d, rank, world, tp, pp, dp, device;
  mp_model_cfg cfg;
  int esz;                       // storage element size
  ncclDataType_t nccl_dt;
  // communicators
  ncclComm_t world_comm = nullptr, tp_comm = nullptr, emb_comm = nullptr;
  ncclComm_t dp_comm = nullptr;   // same (pp, tp) across the d replicas (d > 1): gradient all-reduce at the flush
  // streams
  cudaStream_t cs = nullptr, side = nullptr, s_act_send = nullptr, s_act_recv = nullptr, s_grad_send = nullptr,
               s_grad_recv = nullptr;
  cudaStream_t s_dp = nullptr;   // d > 1: per-layer gradient all-reduces overlapping the last backward passes
  cudaMemPool_t pool = nullptr;
  // stage map
  std::vector<int> dev_of_layer, chunk_of_layer;
  bool has_emb = false, has_head = false;   // stage 0 / stage S-1 on this device
  // parameters (flat)
  std::vector<mp::Param> params;
  std::map<std::string, int> param_index;   // "name#layer" -> index
  std::map<int, mp::LayerParams> layer_params;
  long long n_params = 0;
  float* master = nullptr;     // fp32 master weights
  void* wstore = nullptr;      // storage copy (bf16) or == master (fp32)
  float* grads = nullptr;
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  long long adam_step = 0;
  // stash slots of mp_layer_fwd
  std::map<int, mp::LayerStash> slots;
  int next_slot = 1;
  // workspaces (sized for b = max_b)
  int ws_b = 0;
  void *ws_z = nullptr, *ws_dsq = nullptr, *ws_d4h = nullptr, *ws_dh1 = nullptr, *ws_dh2 = nullptr,
       *ws_dqkv = nullptr, *ws_dctx = nullptr;
  float* ws_fa = nullptr;          // fused-attention backward workspace (dQ accumulator, D)
  float* d_loss = nullptr;
  // deferred logit-layer weight gradient (bf16, last stage): every microbatch's dlogits and
  // final-LN output Z are kept in these row-stacked buffers [m T, V/t] / [m T, h] and
  // dE_r += dlogits^T Z runs once at the flush as one GEMM with K = m T
  void* head_dl = nullptr;
  void* head_z = nullptr;
  size_t head_dl_bytes = 0, head_z_bytes = 0;
  // events for task timing
  std::vector<cudaEvent_t> events;
  int cur_seq0 = 0;                // set by the batch runtime before each microbatch task
  // pipeline channels (p > 1)
  mp::P2PRing p2p;
  // TP-symmetric buffers of the fused g / f all-reduce (t > 1)
  mp::TpSym tps;
};
