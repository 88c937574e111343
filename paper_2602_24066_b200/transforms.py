"""Path transforms feeding the signature path (reference transforms.py:1-52).

``lead_lag`` interleaves each path with its one-step-ahead copy: (B, M+1, d)
samples become (B, 2M+1, 2d), lag channels 0..d-1, lead channels d..2d-1;
even points carry (X_k, X_k), odd points (X_k, X_{k+1}).  ``time_reverse``
flips the sample axis.  Both are data layout only (no arithmetic); a CUDA
tensor stays on its device.
"""

from __future__ import annotations

import numpy as np
import torch

from .exceptions import DomainError
from .signature import PathBatch, _is_tensor, as_path_batch


class LeadLagBatch(PathBatch):
    """A lead-lag transformed PathBatch that remembers the base dimension."""

    def __init__(self, samples, base_d: int, dtype=None):
        super().__init__(samples, dtype=dtype)
        self.base_d = base_d


def lead_lag(paths) -> LeadLagBatch:
    """(B, M+1, d) -> (B, 2M+1, 2d), lag block first, lead block second."""
    paths = as_path_batch(paths)
    if paths.M < 1:
        raise DomainError("lead-lag needs at least one segment")
    x = paths.samples
    d = paths.d
    if _is_tensor(x):
        lag = torch.repeat_interleave(x, 2, dim=1)[:, :-1]      # X0 X0 X1 X1 ... XM
        lead = torch.repeat_interleave(x, 2, dim=1)[:, 1:]      # X0 X1 X1 X2 ... XM
        return LeadLagBatch(torch.cat([lag, lead], dim=2).contiguous(), base_d=d)
    lag = np.repeat(x, 2, axis=1)[:, :-1]
    lead = np.repeat(x, 2, axis=1)[:, 1:]
    return LeadLagBatch(np.ascontiguousarray(np.concatenate([lag, lead], axis=2)), base_d=d)


def time_reverse(paths) -> PathBatch:
    """Reverse the sample order of every path."""
    paths = as_path_batch(paths)
    x = paths.samples
    if _is_tensor(x):
        return PathBatch(torch.flip(x, dims=[1]).contiguous())
    return PathBatch(np.ascontiguousarray(x[:, ::-1]))
