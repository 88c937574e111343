"""Path gradients: the reference's public backward API on the B200 kernels.

Mirrors /root/reference/pkg/src/sigkit/backward.py:32-221.  The numpy
drop-in keeps the reference's contract -- float64 compute and output for any
input dtype (backward.py:166-167), a leading epsilon column of the upstream
ignored (:177-178), optional checkpoint stride (:183-199) -- while the torch
autograd path (autograd.py) keeps the tensor's dtype.  Both run
``sigb_backward`` (csrc/sigb_level.cu): reconstruction of S_{0,t_j} by
exp(-dX_j), reverse-mode through the shared-prefix Horner recursion, and the
telescoping to sample gradients fused in.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .device import resolve_device
from .exceptions import DomainError, ShapeError
from .signature import PathBatch, _is_tensor, as_path_batch, forward_tensor, to_device, to_host
from .wordcodes import Word, decode_word
from .wordset import WordSet


@dataclass
class GradBatch:
    """upstream dL/dS, increment_grads dL/d(dX_j) (B, M, d), path_grads dL/dX_j (B, M+1, d)."""

    upstream: object
    increment_grads: object
    path_grads: object


# -- scalar reference formulas (backward.py:46-127); host-side, for tests ------------


def exp_coeff_grad(delta: Sequence[float], b: Word, channel: int) -> float:
    """d <exp(delta), b> / d delta[channel]."""
    letters = decode_word(b, len(delta))
    total = 0.0
    for r, x in enumerate(letters):
        if x == channel:
            p = 1.0
            for s, y in enumerate(letters):
                if s != r:
                    p *= float(delta[y])
            total += p
    return total / math.factorial(b.length)


def _exp_word(delta, letters) -> float:
    p = 1.0
    for x in letters:
        p *= float(delta[x])
    return p / math.factorial(len(letters))


def left_step(left: np.ndarray, letters: tuple, delta: np.ndarray) -> np.ndarray:
    """Prefix values pulled back one segment: multiply by exp(-delta)."""
    neg = -np.asarray(delta, dtype=np.float64)
    n = len(letters)
    return np.array([sum(left[k] * _exp_word(neg, letters[k:m]) for k in range(m + 1)) for m in range(n + 1)],
                    dtype=np.asarray(left).dtype)


def right_step(right: np.ndarray, letters: tuple, delta: np.ndarray) -> np.ndarray:
    """Suffix values pushed back one segment: multiply by exp(+delta) on the left."""
    delta = np.asarray(delta, dtype=np.float64)
    n = len(letters)
    return np.array([sum(_exp_word(delta, letters[n - m:n - k]) * right[k] for k in range(m + 1))
                     for m in range(n + 1)], dtype=np.asarray(right).dtype)


@dataclass
class ReconstructionState:
    letters: tuple
    left: np.ndarray
    right: np.ndarray

    @classmethod
    def terminal(cls, letters, terminal_left) -> "ReconstructionState":
        right = np.zeros(len(letters) + 1, dtype=np.float64)
        right[0] = 1.0
        return cls(tuple(letters), np.asarray(terminal_left, dtype=np.float64).copy(), right)

    def step_back(self, delta) -> None:
        self.left = left_step(self.left, self.letters, delta)
        self.right = right_step(self.right, self.letters, delta)


def increment_to_sample_grads(increment_grads) -> np.ndarray:
    """dX_j = dInc_j - dInc_{j+1} with one-sided ends (backward.py:130-147).

    Utility on arbitrary arrays; the GPU backward fuses this step.
    """
    g = np.asarray(increment_grads, dtype=np.float64)
    if g.ndim != 3:
        raise ShapeError(f"increment gradients must have shape (B, M, d), got {g.shape}")
    B, M, d = g.shape
    out = np.zeros((B, M + 1, d), dtype=np.float64)
    out[:, 1:] += g
    out[:, :-1] -= g
    return out


# -- batched backward ------------------------------------------------------------------


def backward_tensor(X: torch.Tensor, ws: WordSet, g: torch.Tensor, g_col0: int, stride: int = 0,
                    S: torch.Tensor | None = None, state: torch.Tensor | None = None, want_inc: bool = False):
    """dL/dX (and dL/d(dX)) on the device.  S / state: a forward already done, else recomputed."""
    plan = ws.plan(X.device)
    if S is None and state is None:
        S, state = forward_tensor(X, ws, want_state=True)
    B, L, d = X.shape
    dX = torch.empty_like(X)
    dinc = torch.empty((B, max(L - 1, 0), d), dtype=X.dtype, device=X.device) if want_inc else None
    if plan.prefix_closed:
        plan.backward(X, S, 1 if ws.include_empty else 0, False, g, g_col0, stride, dX, dinc)
    else:
        plan.backward(X, state, 0, True, g, g_col0, stride, dX, dinc)
    return dX, dinc


def signature_backward(paths, ws: WordSet, upstream, threads: int | None = None,
                       checkpoint_stride: int | None = None) -> GradBatch:
    """Path gradients of sum_w upstream[:, w] * S(w), computed in float64 (backward.py:150-221)."""
    paths = as_path_batch(paths)
    is_t = _is_tensor(paths.samples)
    if paths.dtype != np.float64:
        paths = PathBatch(paths.samples, dtype=np.float64)
    if len(ws) < 1:
        raise DomainError("word set has no words to differentiate")
    if ws.d != paths.d:
        raise ShapeError(f"word set has d={ws.d} but paths have {paths.d} channels")
    if _is_tensor(upstream):
        up = upstream.to(torch.float64)
    else:
        up = np.ascontiguousarray(np.asarray(upstream, dtype=np.float64))
    if up.ndim != 2 or up.shape[0] != paths.B:
        raise ShapeError(f"upstream must have shape ({paths.B}, {len(ws)}), got {tuple(up.shape)}")
    g_col0 = 0
    if ws.include_empty and up.shape[1] == len(ws) + 1:
        g_col0 = 1
    elif up.shape[1] != len(ws):
        raise ShapeError(f"upstream must have {len(ws)} word columns, got {up.shape[1]}")
    if checkpoint_stride is not None and checkpoint_stride < 1:
        raise DomainError(f"checkpoint stride must be >= 1, got {checkpoint_stride}")
    dev = resolve_device(paths.samples.device if is_t and paths.samples.is_cuda else None)
    X = to_device(paths.samples, dev)
    stride = int(checkpoint_stride or 0)
    if not is_t and up.nbytes >= _PIPE_MIN_BYTES and paths.B > 1:
        dX, dinc = _backward_host(X, ws, up, g_col0, stride)
        return GradBatch(upstream=np.ascontiguousarray(up[:, g_col0:]), increment_grads=dinc, path_grads=dX)
    G = to_device(up, dev).contiguous()
    dX, dinc = backward_tensor(X, ws, G, g_col0, stride, want_inc=True)
    up_words = up[:, g_col0:]
    if is_t:
        return GradBatch(upstream=up_words, increment_grads=dinc, path_grads=dX)
    return GradBatch(upstream=np.ascontiguousarray(up_words), increment_grads=to_host(dinc),
                     path_grads=to_host(dX))


# a host upstream this large streams in chunks of paths (_backward_host)
_PIPE_MIN_BYTES = 256 << 20
_PIPE_CHUNK_BYTES = 128 << 20


def _backward_host(X: torch.Tensor, ws: WordSet, up: np.ndarray, g_col0: int, stride: int):
    """The numpy drop-in backward in chunks of paths.  The upstream (8 bytes per word and path: the
    drop-in's dominant transfer) is staged chunk by chunk into two pinned buffers while the
    device runs the previous chunk, each chunk's H2D runs on a side stream, and the gradients
    land in pinned host arrays behind the chunk's kernels.  Paths are independent in the
    kernels, so the values are bitwise those of one launch."""
    dev = X.device
    B, L, d = X.shape
    per = max(1, _PIPE_CHUNK_BYTES // max(1, up.shape[1] * up.itemsize))
    up_t = torch.from_numpy(up)
    dX_h = torch.empty((B, L, d), dtype=X.dtype, pin_memory=True)
    dinc_h = torch.empty((B, max(L - 1, 0), d), dtype=X.dtype, pin_memory=True)
    stage = [torch.empty((per, up.shape[1]), dtype=up_t.dtype, pin_memory=True) for _ in range(2)]
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        staged = [None, None]  # events: the H2D out of stage[i] is done (the buffer may be refilled)
        for k, lo in enumerate(range(0, B, per)):
            hi, i = min(B, lo + per), k % 2
            if staged[i] is not None:
                staged[i].synchronize()
            stage[i][: hi - lo].copy_(up_t[lo:hi])  # host: overlaps the device work queued so far
            with torch.cuda.stream(h2d):
                G = torch.empty((hi - lo, up.shape[1]), dtype=X.dtype, device=dev)
                G.copy_(stage[i][: hi - lo], non_blocking=True)
                staged[i] = torch.cuda.Event()
                staged[i].record(h2d)
            main.wait_event(staged[i])
            G.record_stream(main)
            dX, dinc = backward_tensor(X[lo:hi], ws, G, g_col0, stride, want_inc=True)
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                dX_h[lo:hi].copy_(dX, non_blocking=True)
                dinc_h[lo:hi].copy_(dinc, non_blocking=True)
            dX.record_stream(d2h)
            dinc.record_stream(d2h)
        d2h.synchronize()
    return dX_h.numpy(), dinc_h.numpy()
