"""PyTorch autograd over the signature kernels ("autograd backward" of north_star).

``signature(X, ws)`` returns S (B, width) for a CUDA tensor X (B, L, d) and
differentiates through ``sigb_backward``.  Memory-lean: autograd saves only
X and the terminal signature (plus the closure state when the word set is
not prefix-closed) -- no per-step trajectory.
"""

from __future__ import annotations

import torch

from .exceptions import ShapeError
from .gradient import backward_tensor
from .signature import forward_tensor
from .wordset import WordSet


class _SignatureFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X: torch.Tensor, ws: WordSet, stride: int):
        X = X.contiguous()
        out, state = forward_tensor(X, ws, want_state=True)
        ctx.ws = ws
        ctx.stride = stride
        ctx.save_for_backward(X, out, state if state is not None else out)
        ctx.has_state = state is not None
        return out

    @staticmethod
    def backward(ctx, grad_out: torch.Tensor):
        X, out, state = ctx.saved_tensors
        ws = ctx.ws
        g = grad_out.contiguous()
        dX, _ = backward_tensor(X, ws, g, 1 if ws.include_empty else 0, ctx.stride, S=out,
                                state=state if ctx.has_state else None)
        return dX, None, None


def signature(X: torch.Tensor, ws: WordSet, checkpoint_stride: int | None = None) -> torch.Tensor:
    """Differentiable signature coefficients of CUDA paths X (B, L, d) over ``ws``."""
    if not isinstance(X, torch.Tensor) or not X.is_cuda:
        raise ShapeError("signature() takes a CUDA tensor; use signature_forward for numpy input")
    if X.dim() != 3 or X.shape[2] != ws.d:
        raise ShapeError(f"expected (B, L, {ws.d}) paths, got {tuple(X.shape)}")
    if X.dtype not in (torch.float32, torch.float64):
        X = X.to(torch.float64)
    return _SignatureFn.apply(X, ws, int(checkpoint_stride or 0))


class Signature(torch.nn.Module):
    """nn.Module wrapper: ``Signature(ws)(X) -> S``."""

    def __init__(self, ws: WordSet, checkpoint_stride: int | None = None):
        super().__init__()
        self.ws = ws
        self.checkpoint_stride = checkpoint_stride

    def forward(self, X: torch.Tensor) -> torch.Tensor:
        return signature(X, self.ws, self.checkpoint_stride)

    def extra_repr(self) -> str:
        return repr(self.ws)
