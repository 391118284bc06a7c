"""Thin ctypes binding of the C ABI (include/mp.h, include/mp_ops.h).

Argument marshalling only: every step of the path runs in libmp.so.  There is
no fallback -- if the library is missing or cannot be loaded, every call
raises.  Device buffers are passed as integer addresses (e.g. a torch
tensor's data_ptr()); torch is used by callers only for device memory,
streams and process groups.
"""
import ctypes
import os

import numpy as np

# The pipeline runtime uses one compute stream, one side stream and four P2P
# channel streams per process.  A channel stream waits on a peer's slot flag
# with cuStreamWaitValue32 (p2p.cu); with fewer hardware work queues than
# streams that wait can sit in a queue shared with another stream's work and
# block it (false dependency -> deadlock), so ask for the maximum before CUDA
# initialises in this process.  mp_init refuses p > 1 when the setting is
# too small.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libmp.so")

MP_OK, MP_EINVAL, MP_EDIV, MP_EBUDGET, MP_ESCHED, MP_ENOMEM, MP_ECUDA, MP_ENCCL, MP_ESTATE, MP_EUNSUPPORTED = range(10)
STATUS_NAMES = ["MP_OK", "MP_EINVAL", "MP_EDIV", "MP_EBUDGET", "MP_ESCHED", "MP_ENOMEM", "MP_ECUDA",
                "MP_ENCCL", "MP_ESTATE", "MP_EUNSUPPORTED"]
MP_GPIPE, MP_1F1B, MP_INTERLEAVED = 0, 1, 2
SCHEDULES = {"gpipe": MP_GPIPE, "1f1b": MP_1F1B, "interleaved": MP_INTERLEAVED}
MP_FP32, MP_BF16 = 0, 1
DTYPES = {"fp32": MP_FP32, "bf16": MP_BF16}


class MPError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 10 else status}: {msg}")
        self.status = status


class ModelCfg(ctypes.Structure):
    _fields_ = [("l", ctypes.c_int), ("h", ctypes.c_int), ("a", ctypes.c_int), ("s", ctypes.c_int),
                ("V", ctypes.c_int), ("dtype", ctypes.c_int), ("p_drop_attn", ctypes.c_float),
                ("p_drop_hidden", ctypes.c_float), ("ln_eps", ctypes.c_float), ("recompute", ctypes.c_int),
                ("seed", ctypes.c_ulonglong), ("lr", ctypes.c_float), ("attn_impl", ctypes.c_int),
                ("tp_comm", ctypes.c_int)]


class BatchStats(ctypes.Structure):
    _fields_ = [("iter_seconds", ctypes.c_double), ("model_flops", ctypes.c_double),
                ("model_tflops_per_gpu", ctypes.c_double), ("busy_seconds", ctypes.c_double),
                ("bubble_measured", ctypes.c_double), ("bubble_formula", ctypes.c_double),
                ("peak_inflight", ctypes.c_int), ("n_tasks", ctypes.c_int), ("pipeline_seconds", ctypes.c_double),
                ("t_fwd_task", ctypes.c_double), ("t_bwd_task", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GemmDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int), ("batch", ctypes.c_int),
                ("a_major", ctypes.c_int), ("b_major", ctypes.c_int),
                ("A", ctypes.c_void_p), ("lda", ctypes.c_longlong), ("strideA", ctypes.c_longlong),
                ("B", ctypes.c_void_p), ("ldb", ctypes.c_longlong), ("strideB", ctypes.c_longlong),
                ("C", ctypes.c_void_p), ("ldc", ctypes.c_longlong), ("strideC", ctypes.c_longlong),
                ("bias", ctypes.c_void_p), ("c_fp32", ctypes.c_int), ("accumulate", ctypes.c_int),
                ("causal", ctypes.c_int), ("alpha", ctypes.c_float), ("act", ctypes.c_int),
                ("C2", ctypes.c_void_p), ("colsum", ctypes.c_void_p)]


_lib = None
_P, _I, _LL, _F, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_float, ctypes.c_double

# name -> (restype, argtypes); every symbol declared in include/*.h
SIGNATURES = {
    "mp_flops": (_D, [_LL, _LL, _LL, _LL, _LL, _I]),
    "mp_param_count": (ctypes.c_ulonglong, [_LL, _LL, _LL, _LL]),
    "mp_validate": (_I, [ctypes.POINTER(ModelCfg), _I, _I, _I, _I, _I, _I, _I]),
    "mp_get_schedule": (_I, [_I, _I, _I, _I, _I, _P, ctypes.POINTER(_I)]),
    "mp_get_stage_map": (_I, [_I, _I, _I, _P, _P]),
    "mp_bubble_replay": (_I, [_I, _I, _I, _I, _P, _P, _P]),
    "mp_last_error": (ctypes.c_char_p, []),
    "mp_nccl_id_bytes": (_I, []),
    "mp_nccl_get_id": (_I, [_P]),
    "mp_init": (_I, [_I, _I, _I, _I, ctypes.POINTER(ModelCfg), _I, _I, _I, _P, ctypes.POINTER(_P)]),
    "mp_finalize": (_I, [_P]),
    "mp_set_weights": (_I, [_P, ctypes.c_char_p, _I, _P]),
    "mp_set_weights_f64": (_I, [_P, ctypes.c_char_p, _I, _P]),
    "mp_get_weights": (_I, [_P, ctypes.c_char_p, _I, _P, ctypes.POINTER(_LL)]),
    "mp_get_grads": (_I, [_P, ctypes.c_char_p, _I, _P, ctypes.POINTER(_LL)]),
    "mp_zero_grads": (_I, [_P]),
    "mp_layer_fwd": (_I, [_P, _I, _I, _P, _P, ctypes.POINTER(_I), _P]),
    "mp_layer_bwd": (_I, [_P, _I, _I, _I, _P, _P, _P]),
    "mp_head_fwd_bwd": (_I, [_P, _I, _P, _P, _I, _F, _P, _P, _P]),
    "mp_run_batch": (_I, [_P, _I, _I, _I, _I, _P, _I, ctypes.POINTER(_F), ctypes.POINTER(BatchStats)]),
    "mp_compute_stream": (_P, [_P]),
    "mp_tp_comm_mode": (_I, [_P]),
    "mp_tp_reduce_probe": (_I, [_P, _I, _I, ctypes.POINTER(_D)]),
    "mp_run_batch_dev": (_I, [_P, _I, _I, _I, _I, _P, _I, _P, ctypes.POINTER(BatchStats)]),
    "mp_op_gemm": (_I, [_I, ctypes.POINTER(GemmDesc), _P]),
    "mp_gemm_flops": (_D, [ctypes.POINTER(GemmDesc)]),
    "mp_profile_gemm": (_I, [_I]),
    "mp_profile_gemm_read": (_I, [ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_LL)]),
    "mp_launch_count": (_LL, []),
    "mp_op_gemm_config": (_I, [ctypes.POINTER(GemmDesc), _P]),
    "mp_op_layernorm_fwd": (_I, [_I, _P, _P, _P, _P, _P, _P, _I, _I, _F, _P]),
    "mp_op_bda_layernorm_fwd": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _F, _P]),
    "mp_op_layernorm_bwd": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "mp_op_layernorm_bwd_sums": (_I, [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P]),
    "mp_op_bias_gelu_fwd": (_I, [_I, _P, _P, _P, _LL, _I, _P]),
    "mp_op_bias_gelu_bwd": (_I, [_I, _P, _P, _P, _P, _P, _I, _I, _P]),
    "mp_op_softmax_causal_fwd": (_I, [_I, _P, _LL, _I, _F, _P]),
    "mp_op_softmax_causal_bwd": (_I, [_I, _P, _P, _LL, _I, _F, _P]),
    "mp_op_colsum_accum": (_I, [_I, _P, _P, _I, _I, _P]),
    "mp_op_flash_attn_fwd": (_I, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "mp_op_flash_attn_bwd_ws_floats": (_LL, [_I, _I, _I, _I]),
    "mp_op_flash_attn_bwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P]),
}


def lib():
    """Load libmp.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2104_04473_b200.build`")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name, None)
            if f is None:
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st != MP_OK:
        raise MPError(st, lib().mp_last_error().decode())


def _sym(name):
    f = getattr(lib(), name, None)
    if f is None:
        raise MPError(MP_EUNSUPPORTED, f"{name} not exported by {LIB_PATH}")
    return f


# ----------------------------------------------------------------- host-only
def mp_flops(B, s, l, h, V, recompute=True):
    return _sym("mp_flops")(B, s, l, h, V, int(recompute))


def mp_param_count(l, h, s, V):
    return _sym("mp_param_count")(l, h, s, V)


ATTN = {"unfused": 0, "fused": 1}


TP_COMM = {"auto": 0, "nccl": 1, "nvls": 2}


def make_cfg(l, h, a, s, V, dtype="bf16", p_drop_attn=0.0, p_drop_hidden=0.0, ln_eps=1e-5, recompute=False,
             seed=1234, lr=1e-4, attn="unfused", tp_comm="auto"):
    return ModelCfg(l, h, a, s, V, DTYPES[dtype], p_drop_attn, p_drop_hidden, ln_eps, int(recompute), seed, lr,
                    ATTN[attn], TP_COMM[tp_comm])


def mp_validate(cfg, t, p, v, d, B=0, b=1, sched="interleaved"):
    return _sym("mp_validate")(ctypes.byref(cfg), t, p, v, d, B, b, SCHEDULES[sched])


def mp_get_schedule(p, m, v, sched, device):
    n = _I(0)
    _check(_sym("mp_get_schedule")(p, m, v, SCHEDULES[sched], device, None, ctypes.byref(n)))
    buf = (ctypes.c_int * (3 * n.value))()
    _check(_sym("mp_get_schedule")(p, m, v, SCHEDULES[sched], device, buf, ctypes.byref(n)))
    arr = np.frombuffer(buf, dtype=np.int32).reshape(-1, 3)
    return [("F" if k == 0 else "B", int(i), int(c)) for k, i, c in arr]


def mp_get_stage_map(l, p, v):
    dev = (ctypes.c_int * l)()
    ch = (ctypes.c_int * l)()
    _check(_sym("mp_get_stage_map")(l, p, v, dev, ch))
    return list(dev), list(ch)


def mp_bubble_replay(p, m, v, sched, tf, tb):
    """Per-device idle share of the static task orders replayed with task durations
    tf[r], tb[r] and zero communication (host-only, see include/mp.h)."""
    a = (ctypes.c_double * p)(*tf)
    b = (ctypes.c_double * p)(*tb)
    out = (ctypes.c_double * p)()
    _check(_sym("mp_bubble_replay")(p, m, v, SCHEDULES[sched], a, b, out))
    return list(out)


def mp_nccl_get_id():
    n = _sym("mp_nccl_id_bytes")()
    buf = ctypes.create_string_buffer(n)
    _check(_sym("mp_nccl_get_id")(buf))
    return buf.raw


# ------------------------------------------------------------------- ops
def mp_op_gemm(dtype, desc, stream=0):
    _check(_sym("mp_op_gemm")(DTYPES[dtype] if isinstance(dtype, str) else dtype, ctypes.byref(desc), stream))


def mp_op_gemm_config(desc):
    out = (ctypes.c_int * 3)()
    _check(_sym("mp_op_gemm_config")(ctypes.byref(desc), out))
    return tuple(out)


def call(name, *args):
    """Generic marshalling for the mp_op_* kernel entry points (dtype given as
    'bf16' / 'fp32' in the first position)."""
    if args and isinstance(args[0], str):
        args = (DTYPES[args[0]],) + tuple(args[1:])
    _check(_sym(name)(*args))


def raw(name, *args):
    """Call an entry point that returns a value rather than an mp_status."""
    return _sym(name)(*args)


# ----------------------------------------------------------------- context
class Context:
    """Owns an mp_ctx*: mp_init on construction, mp_finalize on close()."""

    def __init__(self, t, p, v, d, cfg, world_rank, world_size, local_device, nccl_id):
        self.cfg = cfg
        self.t, self.p, self.v, self.d = t, p, v, d
        self.ptr = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, len(nccl_id))
        _check(_sym("mp_init")(t, p, v, d, ctypes.byref(cfg), world_rank, world_size, local_device, idbuf,
                                ctypes.byref(self.ptr)))

    def close(self):
        if self.ptr:
            _check(_sym("mp_finalize")(self.ptr))
            self.ptr = ctypes.c_void_p()

    def set_weights(self, name, layer, arr):
        a = np.ascontiguousarray(arr, dtype=np.float32)
        _check(_sym("mp_set_weights")(self.ptr, name.encode(), layer, a.ctypes.data))

    def _get(self, fn, name, layer):
        n = _LL(0)
        _check(_sym(fn)(self.ptr, name.encode(), layer, None, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        _check(_sym(fn)(self.ptr, name.encode(), layer, out.ctypes.data, ctypes.byref(n)))
        return out

    def get_weights(self, name, layer=0):
        return self._get("mp_get_weights", name, layer)

    def get_grads(self, name, layer=0):
        return self._get("mp_get_grads", name, layer)

    def zero_grads(self):
        _check(_sym("mp_zero_grads")(self.ptr))

    def layer_fwd(self, layer, b, x_ptr, y_ptr, stream=0):
        slot = _I(-1)
        _check(_sym("mp_layer_fwd")(self.ptr, layer, b, x_ptr, y_ptr, ctypes.byref(slot), stream))
        return slot.value

    def layer_bwd(self, layer, b, slot, dy_ptr, dx_ptr, stream=0):
        _check(_sym("mp_layer_bwd")(self.ptr, layer, b, slot, dy_ptr, dx_ptr, stream))

    def head_fwd_bwd(self, b, x_ptr, labels_ptr, labels_ld, scale, dx_ptr, loss_ptr, stream=0):
        """Last-stage head (final LN, tied logits, cross-entropy) fwd + bwd; device addresses."""
        _check(_sym("mp_head_fwd_bwd")(self.ptr, b, x_ptr, labels_ptr, labels_ld, scale, dx_ptr, loss_ptr, stream))

    def run_batch(self, B, b, m, sched, tokens, apply_optimizer=False, stats=True):
        """tokens: numpy int32 [B, s+1] or an integer host address (e.g. pinned memory)."""
        if isinstance(tokens, int):
            addr = tokens
        else:
            tok = np.ascontiguousarray(tokens, dtype=np.int32)
            addr = tok.ctypes.data
        loss = _F(0.0)
        st = BatchStats()
        _check(_sym("mp_run_batch")(self.ptr, B, b, m, SCHEDULES[sched], addr, int(apply_optimizer),
                                    ctypes.byref(loss), ctypes.byref(st) if stats else None))
        return loss.value, (st.as_dict() if stats else None)

    def stream(self):
        return _sym("mp_compute_stream")(self.ptr)

    def tp_comm_mode(self):
        """'nccl' / 'nvls' (the transport of the layer all-reduces), 'auto' before the first layer call."""
        return {v: k for k, v in TP_COMM.items()}[_sym("mp_tp_comm_mode")(self.ptr)]

    def tp_reduce_probe(self, b, iters=20):
        """Seconds per fused g / f reduction on the NVLS path (collective over the TP group)."""
        sec = ctypes.c_double()
        _check(_sym("mp_tp_reduce_probe")(self.ptr, b, iters, ctypes.byref(sec)))
        return sec.value

    def run_batch_dev(self, B, b, m, sched, d_tokens, d_loss, apply_optimizer=False, stats=False):
        """Device-resident variant: d_tokens / d_loss are device addresses."""
        st = BatchStats()
        _check(_sym("mp_run_batch_dev")(self.ptr, B, b, m, SCHEDULES[sched], d_tokens, int(apply_optimizer), d_loss,
                                        ctypes.byref(st) if stats else None))
        return st.as_dict() if stats else None


def profile_gemm(enable):
    _check(_sym("mp_profile_gemm")(int(enable)))


def profile_gemm_read():
    f, t, n = _D(0), _D(0), _LL(0)
    _check(_sym("mp_profile_gemm_read")(ctypes.byref(f), ctypes.byref(t), ctypes.byref(n)))
    return f.value, t.value, n.value


def launch_count():
    return _sym("mp_launch_count")()
