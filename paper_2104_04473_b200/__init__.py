"""B200-native (sm_100a) implementation of the PTD-P hot path of
Narayanan et al., arXiv 2104.04473: GPT transformer layer forward/backward
under Megatron tensor parallelism composed with the interleaved 1F1B
pipeline schedule.  The product is the C-ABI library lib/libmp.so
(include/mp.h); `mp` is its thin ctypes binding."""
from . import mp  # noqa: F401
