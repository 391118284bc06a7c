/*
 * mp.h -- C ABI of the B200-native PTD-P hot path (arXiv 2104.04473).
 *
 * Narayanan et al., "Efficient Large-Scale Language Model Training on GPU
 * Clusters Using Megatron-LM" (SC'21).  Citations: P:n = PAPER.md line n.
 *
 * The library computes the forward and backward of GPT transformer layers
 * under Megatron tensor parallelism (Sec. 2.3: column-parallel
 * QKV/FC1, row-parallel projection/FC2, conjugate f/g operators) composed with
 * the pipeline schedules of Sec. 2.2 (GPipe P:104-107, 1F1B P:109,
 * interleaved 1F1B P:112-120), with one process per GPU.  Tensor-parallel
 * reductions use NCCL (ncclAllReduce) or, by default where the NVSwitch offers
 * multicast, NVLS reduce-loads fused into the consuming kernels; pipeline
 * point-to-point transfers use CUDA-IPC receive rings over NVLink written by
 * the copy engine and flagged with stream memory operations (p2p.cu).
 *
 * Conventions
 *  - Every call returns an mp_status; no exceptions or exit() cross the ABI.
 *    mp_last_error() gives a thread-local message for the last failure.
 *  - Indices are 0-based (the paper's figures number microbatches from 1).
 *  - Caller-owned buffers are borrowed for the duration of the call; device
 *    buffers passed to *_fwd/*_bwd calls are used in stream order on the
 *    given CUDA stream (cudaStream_t passed as void*; NULL = legacy stream).
 *  - The library owns weights, gradients, optimizer state, activation stash,
 *    NCCL communicators and internal streams; mp_finalize releases them.
 *  - There is no CPU fallback: compute calls fail with MP_ECUDA when no
 *    sm_100 device is present.  Host-only calls (mp_flops, mp_param_count,
 *    mp_get_schedule, mp_get_stage_map, mp_bubble_replay, mp_validate) need no GPU.
 */
#ifndef MP_H_
#define MP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MP_OK = 0,
  MP_EINVAL = 1,        /* bad argument (null pointer, out-of-range index, unknown name) */
  MP_EDIV = 2,          /* divisibility violated: h%a, a%t, 4h%t, V%t, l%(p*v), t*p*d != world */
  MP_EBUDGET = 3,       /* device memory budget exceeded (S:175 BudgetError) */
  MP_ESCHED = 4,        /* schedule invalid: interleaved needs m % p == 0; v > 1 only for interleaved */
  MP_ENOMEM = 5,        /* allocation failed */
  MP_ECUDA = 6,         /* CUDA error or no usable sm_100 device */
  MP_ENCCL = 7,         /* NCCL error */
  MP_ESTATE = 8,        /* call order (e.g. layer call before mp_set_weights) */
  MP_EUNSUPPORTED = 9   /* valid in the paper but not built here (e.g. NVLS forced without multicast) */
} mp_status;

typedef enum { MP_GPIPE = 0, MP_1F1B = 1, MP_INTERLEAVED = 2 } mp_schedule;
typedef enum { MP_FP32 = 0, MP_BF16 = 1 } mp_dtype;
/* Transport of the layer's g / f all-reduces when t > 1. */
typedef enum {
  MP_TP_COMM_AUTO = 0,   /* NVLS fused when the TP group has NVSwitch multicast, else NCCL */
  MP_TP_COMM_NCCL = 1,   /* the paper's: ncclAllReduce of the partial product, then the elementwise kernel */
  MP_TP_COMM_NVLS = 2    /* required: partials in an NCCL symmetric window, summed by the NVSwitch inside
                            the consuming kernel's loads (multimem.ld_reduce); MP_EUNSUPPORTED if absent */
} mp_tp_comm;

/* GPT model shape (V = 51200, s = 2048 in the paper's models). */
typedef struct {
  int l;                 /* transformer layers */
  int h;                 /* hidden size */
  int a;                 /* attention heads */
  int s;                 /* sequence length */
  int V;                 /* vocabulary size */
  mp_dtype dtype;        /* storage/compute precision of the path (fp32 math inside bf16 kernels) */
  float p_drop_attn;     /* attention-probability dropout (reading #7); 0 = off */
  float p_drop_hidden;   /* hidden dropout after proj / FC2; 0 = off.  Masks are Philox-4x32-10
                            keyed by `seed` and each element's global (sequence, position, feature /
                            head, query, key) coordinates, regenerated in the backward (reading #6) */
  float ln_eps;          /* LayerNorm epsilon (reading #2: 1e-5) */
  int recompute;         /* activation recomputation: mp_run_batch keeps only each layer's
                            input [s, b, h] between a microbatch's forward and backward task and re-runs
                            the layer forward right before its backward (checkpoint every layer); the
                            batch FLOP count becomes Eq. (2)'s 96-formula */
  unsigned long long seed;  /* dropout stream key */
  float lr;              /* Adam learning rate for mp_run_batch(apply_optimizer=1) */
  int attn_impl;         /* 0: the paper's attention core -- strided-batched scores GEMM, fused
                            scale-mask-softmax, P.V GEMM; 1: fused tcgen05 flash kernel
                            (bf16, hd in {32,64,96,128}; otherwise falls back to 0) */
  int tp_comm;           /* mp_tp_comm; the environment variable MP_TP_COMM=nccl overrides AUTO/NVLS */
} mp_model_cfg;

/* Per-batch statistics filled by mp_run_batch. */
typedef struct {
  double iter_seconds;          /* device time of the batch on this rank (events around the whole batch) */
  double model_flops;           /* Eq. (2) F for this batch (72-variant without recompute) */
  double model_tflops_per_gpu;  /* F / (n * iter_seconds) / 1e12 */
  double busy_seconds;          /* sum of this rank's task durations (forward/backward chunk work) */
  double bubble_measured;       /* (pipeline_seconds - busy) / busy on this rank (P:104-105 t_pb / t_id) */
  double bubble_formula;        /* (p-1)/m or (p-1)/(v m) */
  int peak_inflight;            /* max stashed (microbatch, chunk) on this rank */
  int n_tasks;                  /* tasks executed on this rank (2 m v) */
  double pipeline_seconds;      /* batch start -> end of this rank's last task (excludes the flush) */
  double t_fwd_task;            /* mean forward-task (one chunk, one microbatch) duration on this rank */
  double t_bwd_task;            /* mean backward-task duration on this rank */
} mp_batch_stats;

typedef struct mp_ctx mp_ctx;   /* opaque; one per process (= one GPU) */

/* ---------------------------------------------------------------- host-only */

/* Eq. (2): F = 96 B s l h^2 (1 + s/(6h) + V/(16 l h)) when
 * recompute != 0; otherwise 72 B s l h^2 (1 + s/(6h)) + 6 B s h V. */
double mp_flops(long long B, long long s, long long l, long long h, long long V, int recompute);

/* Eq. (1) as the exact integer 12 l h^2 + 13 l h + (V + s) h. */
unsigned long long mp_param_count(long long l, long long h, long long s, long long V);

/* Validate a parallel configuration: returns MP_OK, MP_EDIV,
 * MP_ESCHED or MP_EUNSUPPORTED.  m = B/(b d) is checked when B > 0. */
mp_status mp_validate(const mp_model_cfg* cfg, int t, int p, int v, int d, int B, int b,
                      mp_schedule sched);

/* Per-device task order of a schedule.  `triples` receives
 * 3 * 2*m*v ints: (kind 0 = forward / 1 = backward, microbatch, chunk) in
 * execution order for device `device` in [0, p); *n receives the number of
 * tasks.  `triples` may be NULL to query *n only.  Errors: MP_ESCHED
 * (m % p != 0 for interleaved; v != 1 for GPipe/1F1B), MP_EINVAL. */
mp_status mp_get_schedule(int p, int m, int v, mp_schedule sched, int device, int* triples, int* n);

/* Layer -> (device, chunk) map: stage sigma = chunk * p + device
 * owns layers [sigma L_c, (sigma+1) L_c), L_c = l / (p v).  Output arrays
 * have l entries.  MP_EDIV if l % (p v) != 0. */
mp_status mp_get_stage_map(int l, int p, int v, int* dev_of_layer, int* chunk_of_layer);
/* Ideal-pipeline replay: the static task orders of
 * mp_get_schedule executed with per-device forward / backward task durations
 * tf[r], tb[r] (any unit, p entries each) and zero communication, every task
 * starting when its device is free and its dependency (F(i, s-1); B(i, s+1) or
 * F(i, S-1) on the last stage) has finished.  bubble[r] (p entries, caller-
 * owned) = (end_r - busy_r) / busy_r with busy_r = m v (tf[r] + tb[r]) and
 * end_r the device's last task end, t = 0 at the batch start: equal durations
 * give exactly (p-1)/m (1F1B) or (p-1)/(v m) (interleaved) on device 0; unequal
 * ones show what stage imbalance alone costs.  Host-only, no GPU.  MP_ESTATE if
 * the orders deadlock (never for the library's schedules). */
mp_status mp_bubble_replay(int p, int m, int v, mp_schedule sched, const double* tf, const double* tb,
                           double* bubble);

/* Thread-local description of the last error. */
const char* mp_last_error(void);

/* Size of the NCCL unique id blob mp_init expects (NCCL_UNIQUE_ID_BYTES). */
int mp_nccl_id_bytes(void);
/* Create a new NCCL unique id into `out` (mp_nccl_id_bytes() bytes); rank 0
 * calls this and the launcher broadcasts the bytes to every rank. */
mp_status mp_nccl_get_id(void* out);

/* ---------------------------------------------------------------- context */

/* Collective over n = t*p*d ranks.  Ranks are laid out with
 * tensor parallelism fastest: world_rank = (dp * p + pp) * t + tp.
 * `nccl_id` is the world communicator id from mp_nccl_get_id on rank 0.
 * Validates divisibility (MP_EDIV), sets the CUDA device to local_device,
 * builds the TP communicator, the four directed pipeline channels per rank
 * (activations to / from the neighbours, gradients to / from) and the
 * tied-embedding communicator, allocates this rank's weight shards (bf16 or
 * fp32), fp32 gradient accumulators and fp32 Adam state.  d > 1 (data
 * parallelism) adds a communicator over the d replicas of each
 * (pp, tp) shard; mp_run_batch sums the replicas' gradients with one
 * ncclAllReduce at the pipeline flush. */
mp_status mp_init(int t, int p, int v, int d, const mp_model_cfg* cfg, int world_rank, int world_size,
                  int local_device, const void* nccl_id, mp_ctx** out);
mp_status mp_finalize(mp_ctx* ctx);

/* Weights in the UNPARTITIONED layout of gen/__init__.py, host fp32, row-major,
 * math orientation Y = X W (W_qkv [h, 3h] head-major columns, W_o [h, h],
 * W_1 [h, 4h], W_2 [4h, h]; vectors [n]).  Names: ln1_g ln1_b w_qkv b_qkv w_o
 * b_o ln2_g ln2_b w_1 b_1 w_2 b_2 (per layer, `layer` in [0, l)), and emb
 * pos lnf_g lnf_b (layer ignored).  The library keeps only this rank's shard
 * if this rank owns the layer (MP_OK and no-op otherwise).
 * Values are rounded to the storage dtype. */
mp_status mp_set_weights(mp_ctx* ctx, const char* name, int layer, const float* host);
/* Same with fp64 host data (e.g. the oracle's own arrays): each value is rounded once to
 * fp32 (the master copy), then to the storage type, exactly as mp_set_weights would. */
mp_status mp_set_weights_f64(mp_ctx* ctx, const char* name, int layer, const double* host);
/* Read back this rank's shard of a weight / fp32 gradient accumulator into
 * host fp32 memory, in the shard's math orientation (e.g. W_qkv[:, cols of
 * this rank's heads]).  *n receives the element count; host may be NULL to
 * query the size.  MP_EINVAL if this rank does not own the layer. */
mp_status mp_get_weights(mp_ctx* ctx, const char* name, int layer, float* host, long long* n);
mp_status mp_get_grads(mp_ctx* ctx, const char* name, int layer, float* host, long long* n);
/* Zero all gradient accumulators. */
mp_status mp_zero_grads(mp_ctx* ctx);

/* ----------------------------------------------------------- layer calls */

/* One transformer layer forward on this rank's TP group (collective over the
 * t ranks that share the stage): x, y device [s, b, h] in the storage dtype
 * (the paper's [s, b, a, h] layout).  The activations needed by the
 * backward are stashed in a library-owned slot returned in *stash_slot.
 * Runs on `stream`. */
mp_status mp_layer_fwd(mp_ctx* ctx, int layer, int b, const void* x, void* y, int* stash_slot,
                       void* stream);
/* Backward of a stashed forward: dy -> dx (device [s, b, h]); weight
 * gradients are accumulated (fp32) into the library's accumulators; the
 * stash slot is released.  Collective over the TP group. */
mp_status mp_layer_bwd(mp_ctx* ctx, int layer, int b, int stash_slot, const void* dy, void* dx,
                       void* stream);

/* The model head of the last pipeline stage (stage S-1, reading #12):
 * Z = LN_f(x), logits = Z E_r^T over this rank's vocabulary shard (tied
 * embedding, vocab-parallel over the TP group, readings #10-#11; the logit
 * layer of Eq. (2)), token cross-entropy against `labels`, and its
 * backward.  x, dx: device [s, b, h] in the storage dtype; labels: device
 * int32, the label of position i of sequence j at labels[j * labels_ld + i]
 * (labels_ld >= s; mp_run_batch passes tokens + 1 with labels_ld = s + 1).
 * *loss_dev (device float) receives scale * sum of the b*s token losses;
 * dx = d(that)/dx; scale * d/dE_r, d/dgamma_f, d/dbeta_f are ADDED to the fp32
 * gradient accumulators.  MP_EINVAL on a rank that holds no head (pp != p-1).
 * Collective over the TP group (max / sum-exp / target and dZ all-reduces). */
mp_status mp_head_fwd_bwd(mp_ctx* ctx, int b, const void* x, const int* labels, int labels_ld, float scale,
                          void* dx, float* loss_dev, void* stream);

/* ------------------------------------------------------------- batch call */

/* One training iteration of B sequences under `sched`:
 * m = B/(b d) microbatches of b sequences; tokens host int32 [B, s+1]
 * (inputs tok[:, :s], labels tok[:, 1:]); every rank passes the same tokens;
 * data-parallel replica dp (d > 1) trains on rows [dp B/d, (dp+1) B/d).
 * Executes this rank's static task order (mp_get_schedule) with P2P
 * transfers on FIFO channels, flushes, all-reduces the tied
 * embedding gradient between the first and last stage, and, if
 * apply_optimizer, runs one Adam step (lr from cfg) on every parameter.
 * Gradients are zeroed at the start of the batch.  *loss_out = mean token
 * cross-entropy over the B*s tokens (same value on every rank).  stats may
 * be NULL.  Collective over all ranks. */
mp_status mp_run_batch(mp_ctx* ctx, int B, int b, int m, mp_schedule sched, const int* tokens,
                       int apply_optimizer, float* loss_out, mp_batch_stats* stats);

/* The library's compute stream for this context (cudaStream_t as void*): the
 * stream every forward/backward task of mp_run_batch* is issued on, so that
 * callers can bracket batches with CUDA events on it. */
void* mp_compute_stream(mp_ctx* ctx);

/* NVLink calibration of the fused g / f reduction exactly as the layer
 * runs it on the NVLS path: per repetition the next symmetric buffer, the NVLS barrier
 * (one-shot) or slab reduce-load + multicast store + barrier (two-shot, t >= 4), and
 * the consuming bias-residual kernel that reads the t-way sum of s*b*h elements.
 * Collective over the TP group (every TP rank calls it with the same b, iters).
 * *seconds = time per reduction, CUDA events on the compute stream after 3 warm-up
 * repetitions.  MP_EUNSUPPORTED when t = 1 or the context runs the NCCL path. */
mp_status mp_tp_reduce_probe(mp_ctx* ctx, int b, int iters, double* seconds);

/* Transport the layer's g / f all-reduces use on this rank: MP_TP_COMM_NCCL or
 * MP_TP_COMM_NVLS (decided collectively at the first layer call with t > 1;
 * MP_TP_COMM_AUTO before that; MP_TP_COMM_NCCL when t = 1, no collective). */
int mp_tp_comm_mode(const mp_ctx* ctx);

/* mp_run_batch with the inputs already resident in device memory: d_tokens
 * device int32 [B, s+1]; the mean loss is written (stream-ordered) to the
 * device float *d_loss.  No host synchronisation unless stats != NULL.  Used
 * to time the path without host<->device copies; semantics otherwise equal
 * to mp_run_batch. */
mp_status mp_run_batch_dev(mp_ctx* ctx, int B, int b, int m, mp_schedule sched, const int* d_tokens,
                           int apply_optimizer, float* d_loss, mp_batch_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* MP_H_ */
