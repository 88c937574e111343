"""Forward signatures: the reference's public forward API on the B200 kernels.

Mirrors /root/reference/pkg/src/sigkit/sigcore.py:36-263 (PathBatch,
CoefficientBatch, WindowSpec, signature_forward, signature_windows and the
scalar reference formulas).  numpy in -> numpy out (host buffers are staged
through pinned memory); a CUDA torch tensor in -> tensor values out, on the
tensor's device and stream.  All arithmetic runs in ``sigb_forward`` /
``sigb_windows`` (csrc/sigb_level.cu).
"""

from __future__ import annotations

import functools
import math
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .device import resolve_device
from .exceptions import DomainError, ShapeError, WindowError
from .wordcodes import Word, decode_word
from .wordset import WordSet

SUPPORTED_DTYPES = (np.float64, np.float32)


def _is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


class PathBatch:
    """B paths of M+1 samples in R^d (sigcore.py:36-88); validates like the reference."""

    def __init__(self, samples, dtype=None, allow_nonfinite: bool = False):
        if _is_tensor(samples):
            arr = samples
            if dtype is not None:
                arr = arr.to(torch.float64 if np.dtype(dtype) == np.float64 else torch.float32)
            elif arr.dtype not in (torch.float32, torch.float64):
                arr = arr.to(torch.float64)
            if arr.dim() != 3:
                raise ShapeError(f"samples must have shape (B, M+1, d), got {tuple(arr.shape)}")
            if arr.shape[1] < 1:
                raise ShapeError("paths need at least one sample point")
            if not allow_nonfinite and arr.numel() and not bool(torch.isfinite(arr).all()):
                raise DomainError("samples contain non-finite values; pass allow_nonfinite=True to propagate them")
            self.samples = arr.contiguous()
            return
        arr = np.asarray(samples)
        if dtype is not None:
            arr = arr.astype(dtype, copy=False)
        elif arr.dtype not in SUPPORTED_DTYPES:
            arr = arr.astype(np.float64)
        if arr.dtype not in SUPPORTED_DTYPES:
            raise ShapeError(f"unsupported dtype {arr.dtype}; use float64 or float32")
        if arr.ndim != 3:
            raise ShapeError(f"samples must have shape (B, M+1, d), got {arr.shape}")
        if arr.shape[1] < 1:
            raise ShapeError("paths need at least one sample point")
        if not allow_nonfinite and not np.all(np.isfinite(arr)):
            raise DomainError("samples contain non-finite values; pass allow_nonfinite=True to propagate them")
        self.samples = np.ascontiguousarray(arr)

    @property
    def B(self) -> int:
        return int(self.samples.shape[0])

    @property
    def M(self) -> int:
        return int(self.samples.shape[1]) - 1

    @property
    def d(self) -> int:
        return int(self.samples.shape[2])

    @property
    def dtype(self):
        if _is_tensor(self.samples):
            return np.float64 if self.samples.dtype == torch.float64 else np.float32
        return self.samples.dtype

    @functools.cached_property
    def increments(self):
        s = self.samples
        return s[:, 1:] - s[:, :-1]


def as_path_batch(paths, dtype=None) -> PathBatch:
    return paths if isinstance(paths, PathBatch) else PathBatch(paths, dtype=dtype)


@dataclass
class CoefficientBatch:
    """Signature coefficients over a WordSet; column k is wordset word k (+ leading eps)."""

    wordset: WordSet
    values: object

    def __post_init__(self):
        shape = tuple(self.values.shape)
        if len(shape) != 2 or shape[1] != self.wordset.width:
            raise ShapeError(f"coefficient values must have shape (B, {self.wordset.width}), got {shape}")

    @property
    def B(self) -> int:
        return int(self.values.shape[0])

    @property
    def width(self) -> int:
        return int(self.values.shape[1])

    @property
    def word_values(self):
        return self.values[:, 1:] if self.wordset.include_empty else self.values

    def column_names(self) -> list[str]:
        names = self.wordset.word_strings()
        return ["e"] + names if self.wordset.include_empty else names

    def __array__(self, dtype=None, copy=None):
        v = self.values.cpu().numpy() if _is_tensor(self.values) else self.values
        return np.asarray(v, dtype=dtype)


@dataclass(frozen=True)
class WindowSpec:
    """K windows (l, r) over the sample axis, 0 <= l < r (sigcore.py:138-163)."""

    pairs: np.ndarray

    def __post_init__(self):
        arr = np.ascontiguousarray(np.asarray(self.pairs, dtype=np.int64))
        if arr.ndim != 2 or arr.shape[1] != 2:
            raise WindowError(f"window pairs must have shape (K, 2), got {arr.shape}")
        object.__setattr__(self, "pairs", arr)
        if arr.shape[0] == 0:
            raise WindowError("need at least one window")
        if np.any(arr[:, 0] < 0) or np.any(arr[:, 0] >= arr[:, 1]):
            raise WindowError("windows must satisfy 0 <= l < r")

    @property
    def K(self) -> int:
        return int(self.pairs.shape[0])

    def validate_for(self, M: int) -> None:
        over = self.pairs[:, 1] > M
        if np.any(over):
            l, r = self.pairs[over][0]
            raise WindowError(f"window ({l}, {r}) exceeds the last sample index {M}")


# -- scalar reference formulas (sigcore.py:169-195); host-side, for tests --------------


def segment_exp_coeff(delta: Sequence[float], w: Word) -> float:
    """<exp(delta), w> = prod_j delta[w_j] / |w|!."""
    p = 1.0
    for x in decode_word(w, len(delta)):
        p *= float(delta[x])
    return p / math.factorial(w.length)


def horner_update(prev: Sequence[float], delta: Sequence[float], w: Word) -> float:
    """One Horner-form Chen step for word w from its prefix values prev[0..|w|]."""
    letters = decode_word(w, len(delta))
    n = w.length
    if len(prev) != n + 1:
        raise ShapeError(f"need {n + 1} prefix values, got {len(prev)}")
    h = 0.0
    for k, x in enumerate(letters):
        h = float(delta[x]) / (n - k) * (float(prev[k]) + h)
    return float(prev[n]) + h


# -- batched forward ---------------------------------------------------------------------


def _check_compute(paths: PathBatch, ws: WordSet) -> None:
    if len(ws) < 1:
        raise DomainError("word set has no words to compute")
    if ws.d != paths.d:
        raise ShapeError(f"word set has d={ws.d} but paths have {paths.d} channels")


def to_device(samples, device) -> torch.Tensor:
    """Host numpy -> device tensor through pinned memory (or pass a CUDA tensor through)."""
    if _is_tensor(samples):
        return samples.to(device).contiguous()
    host = torch.from_numpy(np.ascontiguousarray(samples))
    if host.numel() and torch.cuda.is_available():
        host = host.pin_memory()
    return host.to(device, non_blocking=True)


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy.  Large results land in pinned host memory (torch's caching
    host allocator), so the D2H copy runs at full PCIe speed instead of through a
    pageable bounce buffer; the returned array keeps the pinned block alive."""
    if t.is_cuda and t.numel() * t.element_size() >= (1 << 20):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()
    return t.cpu().numpy()


def _scan_segments(plan, ws: WordSet, B: int, M: int) -> int:
    """Segments per path for the parallel-in-time forward, 1 = the sequential sweep.

    The register-resident truncated forward runs one path (or a few) per thread block and
    walks the M steps in order, so a batch smaller than a wave of blocks leaves SMs idle for
    the whole sweep (reference PAPER.md: pathsig does not parallelise over the sequence
    either).  Chen's identity S_{0,T} = S_{0,t_1} (x) S_{t_1,t_2} (x) ... splits each path
    into T windows that run as B*T virtual paths of the windowed kernel; a log2(T)-deep tree
    of truncated tensor products (sigb_tensor_mul, sigcore.py:321-334) joins them.  Used for
    full truncations when the batch fills less than half a wave and the paths are long
    (M >= 4,096: the route's launches cost ~0.3 ms, measured on B200 against 2.3 ms sequential
    at d=4, N=4, B=4, M=20,000 and 10.3 ms -> 0.33 ms at M=100,000; SIGB_SCAN=0 disables,
    SIGB_SCAN=2 forces it for any M >= 64)."""
    mode = os.environ.get("SIGB_SCAN", "1")
    if mode == "0" or not ws.is_full_truncation or M < (64 if mode == "2" else 4096):
        return 1
    ctas = int(_lib.lib().sigb_forward_ctas(plan.handle, B))
    sms = int(_lib.lib().sigb_device_sm_count())
    if ctas <= 0 or sms <= 0 or 2 * ctas >= sms:
        return 1
    T = 1
    while T < 64 and T * 2 <= M // 16 and int(_lib.lib().sigb_forward_ctas(plan.handle, B * T)) < 2 * sms:
        T *= 2
    return T


def _scan_forward(X: torch.Tensor, ws: WordSet, plan, T: int, out: torch.Tensor) -> None:
    """out[:, width] = S_{0,T} of each path as the Chen product of T window signatures."""
    from .logsig import _tmul  # the truncated tensor product kernel (sigb_tensor_mul)

    B, L, d = X.shape
    M = L - 1
    W = len(ws)
    edges = np.linspace(0, M, T + 1).round().astype(np.int64)
    bounds = torch.from_numpy(np.stack([edges[:-1], edges[1:]], axis=1)).to(X.device)
    seg = torch.empty((B, T, W + 1), dtype=X.dtype, device=X.device)
    seg[:, :, 0] = 1.0
    win = torch.empty((B, T, W), dtype=X.dtype, device=X.device)
    plan.windows(X, bounds, win)
    seg[:, :, 1:] = win
    N = ws.max_len
    while seg.shape[1] > 1:  # fixed pairing order: bitwise reproducible
        t = seg.shape[1]
        h = t // 2
        x = seg[:, 0:2 * h:2].reshape(B * h, W + 1).contiguous()
        y = seg[:, 1:2 * h:2].reshape(B * h, W + 1).contiguous()
        z = _tmul(x, y, d, N).view(B, h, W + 1)
        seg = torch.cat([z, seg[:, 2 * h:]], dim=1) if t % 2 else z
    if ws.include_empty:
        out.copy_(seg[:, 0])
    else:
        out.copy_(seg[:, 0, 1:])


def forward_tensor(X: torch.Tensor, ws: WordSet, want_state: bool = False):
    """(out (B, width), closure state or None) for a CUDA tensor X (B, L, d)."""
    plan = ws.plan(X.device)
    B = X.shape[0]
    out = torch.empty((B, ws.width), dtype=X.dtype, device=X.device)
    state = None
    if want_state and not plan.prefix_closed:
        state = torch.empty((B, plan.Wc), dtype=X.dtype, device=X.device)
    T = _scan_segments(plan, ws, B, X.shape[1] - 1) if state is None and B > 0 else 1
    if T > 1:
        with torch.cuda.device(X.device):
            _scan_forward(X.contiguous(), ws, plan, T, out)
        return out, state
    plan.forward(X, out, 1 if ws.include_empty else 0, ws.include_empty, state)
    return out, state


def signature_forward(paths, ws: WordSet, threads: int | None = None) -> CoefficientBatch:
    """Signature coefficients of each path at every word of the set (sigcore.py:227-239).

    ``threads`` is accepted for API compatibility; the GPU grid is fixed by the plan.
    """
    paths = as_path_batch(paths)
    _check_compute(paths, ws)
    if _is_tensor(paths.samples):
        X = paths.samples
        dev = resolve_device(X.device if X.is_cuda else None)
        out, _ = forward_tensor(X.to(dev), ws)
        return CoefficientBatch(ws, out)
    dev = resolve_device()
    X = to_device(paths.samples, dev)
    return CoefficientBatch(ws, _forward_to_host(X, ws))


# host results this large stream back in chunks, each copy under the next chunk's forward
_PIPE_MIN_BYTES = 256 << 20
_PIPE_CHUNK_BYTES = 128 << 20


def _forward_to_host(X: torch.Tensor, ws: WordSet) -> np.ndarray:
    """Forward of a device batch whose coefficients go back to host memory (the numpy drop-in).

    Large results are computed in chunks of paths: chunk k's coefficients copy into one pinned
    host array on a side stream while chunk k+1 computes, so the PCIe transfer (the drop-in's
    bound: 4-8 bytes per word and path) overlaps the kernels.  The chunks take the sequential
    route (the kernels are per path, so the values are bitwise those of one launch)."""
    B, width, es = X.shape[0], ws.width, X.element_size()
    plan = ws.plan(X.device)
    if B < 2 or B * width * es < _PIPE_MIN_BYTES or _scan_segments(plan, ws, B, X.shape[1] - 1) > 1:
        out, _ = forward_tensor(X, ws)
        return to_host(out)
    host = torch.empty((B, width), dtype=X.dtype, pin_memory=True)
    per = max(1, _PIPE_CHUNK_BYTES // (width * es))
    with torch.cuda.device(X.device):
        main = torch.cuda.current_stream(X.device)
        side = torch.cuda.Stream(X.device)
        for lo in range(0, B, per):
            hi = min(B, lo + per)
            out = torch.empty((hi - lo, width), dtype=X.dtype, device=X.device)
            plan.forward(X[lo:hi], out, 1 if ws.include_empty else 0, ws.include_empty, None)
            ready = torch.cuda.Event()
            ready.record(main)
            with torch.cuda.stream(side):
                side.wait_event(ready)
                host[lo:hi].copy_(out, non_blocking=True)
            out.record_stream(side)
        side.synchronize()
    return host.numpy()


def signature_windows(paths, ws: WordSet, windows, threads: int | None = None) -> list[CoefficientBatch]:
    """Independent signatures of K sample windows (sigcore.py:242-263)."""
    paths = as_path_batch(paths)
    _check_compute(paths, ws)
    if not isinstance(windows, WindowSpec):
        windows = WindowSpec(np.asarray(windows))
    windows.validate_for(paths.M)
    is_t = _is_tensor(paths.samples)
    dev = resolve_device(paths.samples.device if is_t and paths.samples.is_cuda else None)
    X = to_device(paths.samples, dev)
    bounds = torch.from_numpy(windows.pairs).to(dev)
    plan = ws.plan(dev)
    out = torch.empty((paths.B, windows.K, len(ws)), dtype=X.dtype, device=dev)
    plan.windows(X, bounds, out)
    res = []
    for k in range(windows.K):
        v = out[:, k, :]
        if ws.include_empty:
            v = torch.cat([torch.ones((paths.B, 1), dtype=X.dtype, device=dev), v], dim=1)
        res.append(CoefficientBatch(ws, v if is_t else to_host(v.contiguous())))
    return res
