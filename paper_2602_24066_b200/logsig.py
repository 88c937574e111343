"""Log-signatures and the dense truncated tensor algebra on the B200 kernels.

Mirrors /root/reference/pkg/src/sigkit/logsig.py (LogCoefficientBatch,
tensor_log, tensor_exp, logsignature_forward, logsignature_backward) and the
truncated tensor operations of sigcore.py:266-352 (chen_concat,
signature_inverse).  Same names, argument meaning and errors.

The log-signature routes through the hot path exactly as the reference does:
the signature over the reduced set cl = (all words of length <= N-1) u
(Lyndon words of length N) comes from ``sigb_forward``; the truncated log
series restricted to Lyndon words is a polynomial in those coefficients,
evaluated by ``sigb_logsig_forward`` (its gradient by ``sigb_logsig_backward``,
chained into ``sigb_backward``).  The dense operations are Horner loops of
``sigb_tensor_mul`` (graded product, scale, + unit).
"""

from __future__ import annotations

import functools

import numpy as np
import torch

from . import _lib
from .device import dtype_code, ptr, resolve_device, stream_ptr
from .exceptions import DomainError, ShapeError, UnsupportedWordSetError
from .gradient import GradBatch, backward_tensor
from .signature import CoefficientBatch, PathBatch, _is_tensor, as_path_batch, forward_tensor, to_device, to_host
from .wordset import WordSet, build_lyndon, build_truncated

__all__ = [
    "LogCoefficientBatch", "chen_concat", "logsignature_backward", "logsignature_forward", "signature_inverse",
    "tensor_exp", "tensor_log",
]


class LogCoefficientBatch(CoefficientBatch):
    """Log-signature coefficients over a Lyndon word set (logsig.py:37-38)."""


def _series_coef(k: int) -> float:
    """Coefficient of x^k in log(1 + x)."""
    return (1.0 if k % 2 else -1.0) / k


# -- dense truncated tensors ----------------------------------------------------------


def _depth(ws: WordSet) -> int:
    if not ws.is_full_truncation:
        raise UnsupportedWordSetError(
            "this operation needs a fully truncated word set (all words of "
            f"length 1..N); got kind={ws.kind!r} with {len(ws)} words"
        )
    return ws.max_len


def _dense(a: CoefficientBatch, dev) -> torch.Tensor:
    """Epsilon-first dense layout on the device, epsilon coefficient 1 (sigcore.py:282-288)."""
    v = a.word_values
    t = v.to(dev) if _is_tensor(v) else to_device(np.ascontiguousarray(v), dev)
    one = torch.ones((t.shape[0], 1), dtype=t.dtype, device=dev)
    return torch.cat([one, t], dim=1).contiguous()


def _result(ws: WordSet, full: torch.Tensor, like) -> CoefficientBatch:
    vals = full if ws.include_empty else full[:, 1:]
    vals = vals.contiguous()
    return CoefficientBatch(ws, vals if _is_tensor(like) else to_host(vals))


def _tmul(x: torch.Tensor, y: torch.Tensor, d: int, N: int, scale: float = 1.0, add0: float = 0.0) -> torch.Tensor:
    out = torch.empty_like(x)
    with torch.cuda.device(x.device):  # the ABI launches on the calling thread's current device
        _lib.check(_lib.lib().sigb_tensor_mul(dtype_code(x.dtype), ptr(x), ptr(y), x.shape[0], d, N, float(scale),
                                              float(add0), ptr(out), stream_ptr(x.device)))
    return out


def _unit_like(x: torch.Tensor, value: float) -> torch.Tensor:
    P = torch.zeros_like(x)
    P[:, 0] = value
    return P


def tensor_log(a: CoefficientBatch) -> CoefficientBatch:
    """Truncated tensor logarithm, log(1 + x) = sum_k (-1)^(k+1) x^k / k in Horner form (logsig.py:42-56)."""
    N = _depth(a.wordset)
    d = a.wordset.d
    dev = resolve_device(a.values.device if _is_tensor(a.values) and a.values.is_cuda else None)
    x = _dense(a, dev)
    x[:, 0] = 0.0
    P = _unit_like(x, _series_coef(N))
    for k in range(N - 1, 0, -1):
        P = _tmul(x, P, d, N, 1.0, _series_coef(k))
    out = _tmul(x, P, d, N)
    return _result(a.wordset.with_include_empty(False), out, a.values)


def tensor_exp(a: CoefficientBatch) -> CoefficientBatch:
    """Truncated tensor exponential, the inverse of tensor_log on its image (logsig.py:59-72)."""
    N = _depth(a.wordset)
    d = a.wordset.d
    dev = resolve_device(a.values.device if _is_tensor(a.values) and a.values.is_cuda else None)
    x = _dense(a, dev)
    x[:, 0] = 0.0
    P = _unit_like(x, 1.0)
    for k in range(N, 0, -1):
        P = _tmul(x, P, d, N, 1.0 / k, 1.0)
    return _result(a.wordset.with_include_empty(False), P, a.values)


def chen_concat(a: CoefficientBatch, b: CoefficientBatch) -> CoefficientBatch:
    """Chen product sum_{w = u v} a(u) b(v) over one truncated set (sigcore.py:321-334)."""
    N = _depth(a.wordset)
    if a.wordset != b.wordset:
        raise UnsupportedWordSetError("operands must share one truncated word set")
    if a.B != b.B:
        raise ShapeError(f"batch sizes differ: {a.B} vs {b.B}")
    dev = resolve_device(a.values.device if _is_tensor(a.values) and a.values.is_cuda else None)
    x, y = _dense(a, dev), _dense(b, dev)
    if y.dtype != x.dtype:
        y = y.to(x.dtype)
    return _result(a.wordset, _tmul(x, y, a.wordset.d, N), a.values)


def signature_inverse(a: CoefficientBatch) -> CoefficientBatch:
    """Group inverse by the Neumann series inv <- 1 - x inv, N times (sigcore.py:337-352)."""
    N = _depth(a.wordset)
    d = a.wordset.d
    dev = resolve_device(a.values.device if _is_tensor(a.values) and a.values.is_cuda else None)
    x = _dense(a, dev)
    x[:, 0] = 0.0
    inv = _unit_like(x, 1.0)
    for _ in range(N):
        inv = _tmul(x, inv, d, N, -1.0, 1.0)
    return _result(a.wordset, inv, a.values)


# -- log-signature polynomial ---------------------------------------------------------------


class _Projection:
    """Reduced compute set, Lyndon set and the log-series term tables (logsig.py:79-127)."""

    def __init__(self, d: int, N: int):
        self.lyndon = build_lyndon(d, min(N, 1) if d == 1 else N)
        pairs = set()
        if N >= 2:
            lower = build_truncated(d, N - 1)
            pairs.update(zip(lower.lengths.tolist(), lower.codes.tolist()))
        pairs.update(zip(self.lyndon.lengths.tolist(), self.lyndon.codes.tolist()))
        pairs = sorted(pairs)
        self.compute = WordSet(d, np.array([n for n, _ in pairs], dtype=np.int64),
                               np.array([c for _, c in pairs], dtype=np.uint64), kind="custom",
                               meta={"role": "logsig-internal", "depth": N})
        col = self.compute.global_index
        F = max(int(self.lyndon.max_len), 1)
        term_off, cols, coef, word = [0], [], [], []
        for wi in range(len(self.lyndon)):
            n = int(self.lyndon.lengths[wi])
            code = int(self.lyndon.codes[wi])
            letters = [(code // d ** (n - 1 - k)) % d for k in range(n)]
            # every split of the word into contiguous factors: bit k of `cuts` cuts after letter k
            for cuts in sorted(range(1 << (n - 1)), key=lambda m: (bin(m).count("1"), _cut_order(m, n))):
                bounds = [0] + [k + 1 for k in range(n - 1) if cuts >> k & 1] + [n]
                row = []
                for s, e in zip(bounds[:-1], bounds[1:]):
                    c = 0
                    for x in letters[s:e]:
                        c = c * d + x
                    row.append(col[(e - s, c)])
                coef.append(_series_coef(len(row)))
                cols.append(row + [-1] * (F - len(row)))
                word.append(wi)
            term_off.append(len(coef))
        self.F = F
        self.term_off = np.asarray(term_off, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int32).reshape(-1, F)
        self.coef = np.asarray(coef, dtype=np.float64)
        self.term_word = np.asarray(word, dtype=np.int64)
        # column -> (term, factor) entries, term-major: the gradient gathers in a fixed order
        ents = [[] for _ in range(len(self.compute))]
        for t in range(self.cols.shape[0]):
            for k in range(F):
                c = int(self.cols[t, k])
                if c >= 0:
                    ents[c].append((t << 8) | k)
        self.col_off = np.cumsum([0] + [len(e) for e in ents]).astype(np.int64)
        self.entries = np.asarray([x for e in ents for x in e], dtype=np.int64)
        self._dev = {}

    def device_tables(self, dev):
        key = dev.index
        if key not in self._dev:
            self._dev[key] = {k: torch.from_numpy(getattr(self, k)).to(dev)
                              for k in ("term_off", "cols", "coef", "term_word", "col_off", "entries")}
        return self._dev[key]


def _cut_order(mask: int, n: int) -> tuple:
    """Lexicographic order of the cut positions (the reference's itertools.combinations order)."""
    return tuple(k for k in range(n - 1) if mask >> k & 1)


@functools.lru_cache(maxsize=32)
def _projection(d: int, N: int) -> _Projection:
    return _Projection(d, N)


def _check(paths, d: int, N: int):
    if N < 1:
        raise DomainError(f"depth must be >= 1, got {N}")
    if paths.d != d:
        raise ShapeError(f"paths have {paths.d} channels, expected {d}")


def logsig_tensor(X: torch.Tensor, d: int, N: int) -> torch.Tensor:
    """Lyndon log-signature (B, |Lyndon|) of CUDA samples X (B, L, d)."""
    pr = _projection(d, N)
    S, _ = forward_tensor(X, pr.compute)
    tb = pr.device_tables(X.device)
    out = torch.empty((X.shape[0], len(pr.lyndon)), dtype=X.dtype, device=X.device)
    with torch.cuda.device(X.device):
        _lib.check(_lib.lib().sigb_logsig_forward(dtype_code(X.dtype), ptr(S), S.shape[0], S.shape[1],
                                                  ptr(tb["term_off"]), ptr(tb["cols"]), ptr(tb["coef"]),
                                                  out.shape[1], pr.F, ptr(out), out.shape[1], stream_ptr(X.device)))
    return out


def logsignature_forward(paths, d: int, N: int, threads: int | None = None) -> LogCoefficientBatch:
    """Log-signature coefficients at the Lyndon words of length <= N (logsig.py:139-161)."""
    if N < 1:
        raise DomainError(f"depth must be >= 1, got {N}")
    paths = as_path_batch(paths)
    _check(paths, d, N)
    pr = _projection(d, N)
    is_t = _is_tensor(paths.samples)
    dev = resolve_device(paths.samples.device if is_t and paths.samples.is_cuda else None)
    X = to_device(paths.samples, dev)
    out = logsig_tensor(X, d, N)
    return LogCoefficientBatch(pr.lyndon, out if is_t else to_host(out))


def logsignature_backward(paths, d: int, N: int, grad_out, threads: int | None = None) -> GradBatch:
    """Path gradients of sum_i grad_out[:, i] * logsig_i, in float64 (logsig.py:164-192)."""
    if N < 1:
        raise DomainError(f"depth must be >= 1, got {N}")
    paths = as_path_batch(paths, dtype=np.float64)
    if paths.dtype != np.float64:
        # an existing PathBatch (e.g. lead_lag of float32 samples) is passed through
        # unchanged by as_path_batch; the reference computes this backward in float64
        paths = PathBatch(paths.samples, dtype=np.float64)
    _check(paths, d, N)
    pr = _projection(d, N)
    is_t = _is_tensor(paths.samples)
    g = grad_out.to(torch.float64) if _is_tensor(grad_out) else np.asarray(grad_out, dtype=np.float64)
    if tuple(g.shape) != (paths.B, len(pr.lyndon)):
        raise ShapeError(f"grad_out must have shape ({paths.B}, {len(pr.lyndon)}), got {tuple(g.shape)}")
    dev = resolve_device(paths.samples.device if is_t and paths.samples.is_cuda else None)
    X = to_device(paths.samples, dev)
    G = to_device(g, dev).contiguous()
    S, _ = forward_tensor(X, pr.compute)
    tb = pr.device_tables(dev)
    up = torch.empty_like(S)
    if not (X.dtype == S.dtype == G.dtype == up.dtype == torch.float64):
        raise DomainError(f"log-signature backward runs in float64, got X {X.dtype}, S {S.dtype}, G {G.dtype}")
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().sigb_logsig_backward(
            dtype_code(S.dtype), ptr(S), S.shape[0], S.shape[1], ptr(G), G.shape[1], ptr(tb["col_off"]),
            ptr(tb["entries"]), ptr(tb["term_word"]), ptr(tb["cols"]), ptr(tb["coef"]), pr.F, up.shape[1], ptr(up),
            up.shape[1], stream_ptr(dev)))
    dX, dinc = backward_tensor(X, pr.compute, up, 0, S=S, want_inc=True)
    if is_t:
        return GradBatch(upstream=G, increment_grads=dinc, path_grads=dX)
    return GradBatch(upstream=np.ascontiguousarray(g), increment_grads=to_host(dinc), path_grads=to_host(dX))
