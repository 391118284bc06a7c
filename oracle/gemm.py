"""Plain definition of the (strided-)batched GEMM the hot path is built from
(oracle; test infrastructure only).

Appendix: an A_{m x k} X_{k x n} product costs 2mkn FLOPs; every
linear layer and both attention products ("strided batched
GEMM kernels") are instances of C_z = alpha A_z B_z + bias, here in fp64.
The causal variants restate what the result must be where it is defined:
tiles strictly above the diagonal of a causal score matrix are not part of the
method's output ("implicit causal masking").
"""
import numpy as np


def gemm_ref(A, B, alpha=1.0, bias=None):
    """A [z, M, K], B [z, K, N] -> alpha * A @ B (+ bias[N]) in fp64."""
    C = alpha * np.matmul(np.asarray(A, np.float64), np.asarray(B, np.float64))
    if bias is not None:
        C = C + np.asarray(bias, np.float64)
    return C
