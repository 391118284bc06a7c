"""Helpers for the GPU parity tests: move oracle-layout numpy data to device
tensors of the storage dtype and compare with the normwise metric
max|x - ref| / max|ref| (reading #20)."""
import numpy as np
import torch

import gen


def dev(x, dtype):
    """numpy (already rounded to `dtype`) -> cuda tensor of the storage dtype."""
    t = torch.tensor(np.asarray(x, dtype=np.float32))
    return (t.to(torch.bfloat16) if dtype == "bf16" else t).cuda()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def normwise(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


TOL = {"bf16": 2e-2, "fp32": 1e-4}   # north_star tolerances
