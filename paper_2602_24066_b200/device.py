"""Device plumbing: CUDA device resolution, plans, and raw C-ABI calls.

PyTorch is used only for device memory, streams and pointers; every
computation is one of the sm_100a kernels behind include/sigkit_b200.h.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .exceptions import DomainError


def resolve_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2602_24066_b200 computes on a CUDA device (sm_100a) and there is none; "
            "no CPU fallback exists"
        )
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device; no CPU fallback exists")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def dtype_code(dt) -> int:
    if dt in (torch.float32, np.float32):
        return _lib.SIGB_F32
    if dt in (torch.float64, np.float64):
        return _lib.SIGB_F64
    raise DomainError(f"unsupported dtype {dt}; use float64 or float32")


def wordset_tables(codes: np.ndarray, lengths: np.ndarray, d: int, device=None) -> dict:
    """Run sigb_wordset_tables on the device; returns host numpy copies."""
    dev = resolve_device(device)
    W = int(lengths.size)
    max_len = int(lengths.max()) if W else 0
    L = _lib.lib()
    with torch.cuda.device(dev):
        c = torch.from_numpy(codes.view(np.int64).copy()).to(dev)
        n = torch.from_numpy(np.ascontiguousarray(lengths, dtype=np.int64)).to(dev)
        letters = torch.empty((W, max_len), dtype=torch.int64, device=dev)
        prefix = torch.empty((W, max_len + 1), dtype=torch.int64, device=dev)
        suffix = torch.empty((W, max_len + 1), dtype=torch.int64, device=dev)
        level = torch.empty(max_len + 2, dtype=torch.int64, device=dev)
        bits = max(1, (d - 1).bit_length())
        packed = torch.empty(W, dtype=torch.int64, device=dev) if bits * max_len <= 64 else None
        _lib.check(L.sigb_wordset_tables(ptr(c), ptr(n), W, d, max_len, ptr(letters), ptr(prefix), ptr(suffix),
                                         ptr(level), ptr(packed), stream_ptr(dev)))
        out = {
            "letters": letters.cpu().numpy(),
            "prefix": prefix.cpu().numpy(),
            "suffix": suffix.cpu().numpy(),
            "level_start": level.cpu().numpy(),
        }
        if packed is not None:
            out["packed"] = packed.cpu().numpy().view(np.uint64)
    return out


class Plan:
    """sigb_plan handle of a WordSet on one device (closure + trie schedule)."""

    def __init__(self, ws, device: torch.device):
        self.device = device
        self.d = ws.d
        self.W = len(ws)
        self.include_empty = ws.include_empty
        L = _lib.lib()
        h = ctypes.c_void_p()
        codes = np.ascontiguousarray(ws.codes, dtype=np.uint64)
        lengths = np.ascontiguousarray(ws.lengths, dtype=np.int64)
        with torch.cuda.device(device):
            _lib.check(L.sigb_plan_create(codes.ctypes.data_as(ctypes.c_void_p),
                                          lengths.ctypes.data_as(ctypes.c_void_p), self.W, self.d,
                                          ctypes.byref(h), stream_ptr(device)))
        self.handle = h
        self.Wc = int(L.sigb_plan_closure_size(h))
        self.num_parts = int(L.sigb_plan_num_parts(h))
        self.step_fmas = int(L.sigb_plan_step_fmas(h))
        self.prefix_closed = self.Wc == self.W

    @property
    def kernel_kind(self) -> int:
        """1 truncated, 2 fragment, 4 generated, 0 level-synchronous kernels (current policy)."""
        return int(_lib.lib().sigb_plan_kernel_kind(self.handle))

    @property
    def uses_truncated(self) -> bool:
        return self.kernel_kind == 1

    @property
    def uses_fragments(self) -> bool:
        return self.kernel_kind == 2

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                with torch.cuda.device(self.device):
                    torch.cuda.synchronize(self.device)
                    _lib.lib().sigb_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- raw launches (tensors already on self.device, contiguous) ------------------
    def forward(self, X: torch.Tensor, out: torch.Tensor, out_col0: int, include_empty: bool,
                state: torch.Tensor | None = None) -> None:
        B, L, _ = X.shape
        _lib.check(_lib.lib().sigb_forward(self.handle, dtype_code(X.dtype), ptr(X), B, L, ptr(out),
                                           out.shape[1], out_col0, int(include_empty), ptr(state),
                                           stream_ptr(self.device)))

    def windows(self, X: torch.Tensor, bounds: torch.Tensor, out: torch.Tensor) -> None:
        B, L, _ = X.shape
        _lib.check(_lib.lib().sigb_windows(self.handle, dtype_code(X.dtype), ptr(X), B, L, ptr(bounds),
                                           bounds.shape[0], ptr(out), stream_ptr(self.device)))

    def workspace_bytes(self, dtype, B: int, L: int, stride: int) -> int:
        n = ctypes.c_size_t()
        _lib.check(_lib.lib().sigb_backward_workspace_size(self.handle, dtype_code(dtype), B, L, stride,
                                                           ctypes.byref(n)))
        return int(n.value)

    def backward(self, X: torch.Tensor, S: torch.Tensor, s_col0: int, s_is_state: bool, g: torch.Tensor,
                 g_col0: int, stride: int, dX: torch.Tensor, dinc: torch.Tensor | None = None,
                 work: torch.Tensor | None = None) -> None:
        B, L, _ = X.shape
        nbytes = self.workspace_bytes(X.dtype, B, L, stride)
        if work is None or work.numel() < nbytes:
            work = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=self.device)
        _lib.check(_lib.lib().sigb_backward(self.handle, dtype_code(X.dtype), ptr(X), B, L, ptr(S), S.shape[1],
                                            s_col0, int(s_is_state), ptr(g), g.shape[1], g_col0, stride,
                                            ptr(work), nbytes, ptr(dX), ptr(dinc), stream_ptr(self.device)))
