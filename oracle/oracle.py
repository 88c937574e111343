"""CPU oracle for the signature hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  It wraps
``sig_oracle.c`` (a line-by-line restatement of the reference numba kernels,
see that file's header for the file:line map) through ctypes and adds the two
pure-Python oracles the reference test-suite itself relies on:

* ``dense_signature`` -- level-by-level dense tensor products, restating
  ``testkit.dense_signature_oracle`` (/root/reference/pkg/src/sigkit/testkit.py:45-68);
* ``finite_difference_grad`` -- central differences with step h*max(1,|x|),
  restating ``testkit.finite_difference_grad`` (testkit.py:102-130).

Parity is pinned: ``tests/test_oracle_golden.py`` checks every routine here
against golden vectors produced by importing the reference package itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libsigoracle.so")
_lib = None


def build() -> str:
    """Compile sig_oracle.c with gcc (OpenMP) into oracle/build/."""
    os.makedirs(os.path.join(_HERE, "build"), exist_ok=True)
    src = os.path.join(_HERE, "sig_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-fopenmp", "-std=c11", "-shared", "-o", _SO, src]
        )
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = ctypes.CDLL(_SO)
        _setup(_lib)
    return _lib


_P = ctypes.c_void_p
_I = ctypes.c_int64


def _setup(L):
    sig = {
        "ora_increments_f64": [_P, _I, _I, _I, _P],
        "ora_increments_f32": [_P, _I, _I, _I, _P],
        "ora_letters": [_P, _P, _I, _I, _I, _P],
        "ora_factor_table": [_P, _P, _I, _I, _I, ctypes.c_int, _P],
        "ora_forward_f64": [_P, _I, _I, _I, _P, _P, _I, _I, _P],
        "ora_forward_f32": [_P, _I, _I, _I, _P, _P, _I, _I, _P],
        "ora_windows_f64": [_P, _I, _I, _I, _P, _P, _I, _I, _P, _I, _P],
        "ora_windows_f32": [_P, _I, _I, _I, _P, _P, _I, _I, _P, _I, _P],
        "ora_backward_f64": [_P, _I, _I, _I, _P, _P, _I, _I, _P, _I, _P],
        "ora_sample_grads": [_P, _I, _I, _I, _P],
    }
    for name, argtypes in sig.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = None


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    """Cap the OpenMP pool (the oracle's analogue of sigkit's threads=)."""
    omp = ctypes.CDLL("libgomp.so.1")
    omp.omp_set_num_threads(int(n))


# -- word-set tables (wordsets.py:176-228) -------------------------------------


def letters(codes, lengths, d):
    codes = np.ascontiguousarray(codes, dtype=np.uint64)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    W = lengths.size
    max_len = int(lengths.max()) if W else 0
    out = np.zeros((W, max_len), dtype=np.int64)
    lib().ora_letters(_ptr(codes), _ptr(lengths), W, d, max_len, _ptr(out))
    return out


def factor_table(codes, lengths, d, suffix: bool):
    codes = np.ascontiguousarray(codes, dtype=np.uint64)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    W = lengths.size
    max_len = int(lengths.max()) if W else 0
    out = np.empty((W, max_len + 1), dtype=np.int64)
    lib().ora_factor_table(_ptr(codes), _ptr(lengths), W, d, max_len, int(suffix), _ptr(out))
    return out


def level_offsets(lengths, max_len=None):
    """Start offset of each level 1..max_len+1 in canonical order (wordsets.py:230-247)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    if max_len is None:
        max_len = int(lengths.max()) if lengths.size else 0
    counts = np.bincount(lengths, minlength=max_len + 1)
    return np.concatenate([[0], np.cumsum(counts[1:])]).astype(np.int64)


# -- forward / windows / backward (_kernels.py) ------------------------------------


def increments(X):
    X = np.ascontiguousarray(X)
    B, L, d = X.shape
    out = np.empty((B, max(L - 1, 0), d), dtype=X.dtype)
    fn = lib().ora_increments_f64 if X.dtype == np.float64 else lib().ora_increments_f32
    fn(_ptr(X), B, L, d, _ptr(out))
    return out


def forward(X, codes, lengths, d):
    """Reference forward_kernel over the words (codes, lengths); X (B, L, d) f32|f64."""
    X = np.ascontiguousarray(X)
    assert X.dtype in (np.float32, np.float64)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    lt = letters(codes, lengths, d)
    incr = increments(X)
    B, M = incr.shape[0], incr.shape[1]
    W, max_len = lt.shape
    out = np.empty((B, W), dtype=X.dtype)
    fn = lib().ora_forward_f64 if X.dtype == np.float64 else lib().ora_forward_f32
    fn(_ptr(incr), B, M, d, _ptr(lt), _ptr(lengths), W, max_len, _ptr(out))
    return out


def windows(X, codes, lengths, d, bounds):
    X = np.ascontiguousarray(X)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    lt = letters(codes, lengths, d)
    incr = increments(X)
    B, M = incr.shape[0], incr.shape[1]
    W, max_len = lt.shape
    K = bounds.shape[0]
    out = np.empty((B, K, W), dtype=X.dtype)
    fn = lib().ora_windows_f64 if X.dtype == np.float64 else lib().ora_windows_f32
    fn(_ptr(incr), B, M, d, _ptr(lt), _ptr(lengths), W, max_len, _ptr(bounds), K, _ptr(out))
    return out


def backward(X, codes, lengths, d, upstream, stride: int = 0):
    """Reference backward_kernel + increment_to_sample_grads, float64.

    Returns (increment_grads (B, M, d), path_grads (B, L, d)).
    """
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    up = np.ascontiguousarray(np.asarray(upstream, dtype=np.float64))
    lt = letters(codes, lengths, d)
    incr = increments(X)
    B, M = incr.shape[0], incr.shape[1]
    W, max_len = lt.shape
    ig = np.zeros((B, M, d), dtype=np.float64)
    lib().ora_backward_f64(_ptr(incr), B, M, d, _ptr(lt), _ptr(lengths), W, max_len, _ptr(up),
                           int(stride), _ptr(ig))
    pg = np.empty((B, M + 1, d), dtype=np.float64)
    lib().ora_sample_grads(_ptr(ig), B, M, d, _ptr(pg))
    return ig, pg


# -- independent dense oracles (testkit.py:45-68, :102-130) ------------------------


def _dense_exp(delta, N):
    levels = [np.ones((), dtype=np.float64)]
    for n in range(1, N + 1):
        levels.append(np.multiply.outer(levels[-1], delta) / n)
    return levels


def _dense_mul(a, b, N):
    out = []
    for n in range(N + 1):
        acc = np.zeros((a[1].shape[0],) * n, dtype=np.float64)
        for m in range(n + 1):
            acc += np.multiply.outer(a[m], b[n - m])
        out.append(acc)
    return out


def dense_signature(X, d, N):
    """All words of length 1..N in canonical order, by dense tensor products (fp64)."""
    X = np.asarray(X, dtype=np.float64)
    B = X.shape[0]
    width = sum(d**n for n in range(1, N + 1))
    out = np.empty((B, width), dtype=np.float64)
    for b in range(B):
        sig = _dense_exp(np.zeros(d), N)
        for j in range(X.shape[1] - 1):
            sig = _dense_mul(sig, _dense_exp(X[b, j + 1] - X[b, j], N), N)
        out[b] = np.concatenate([sig[n].reshape(-1) for n in range(1, N + 1)])
    return out


def dense_columns(codes, lengths, d, dense_values):
    """Columns of a dense_signature result matching arbitrary (codes, lengths)."""
    offsets = {1: 0}
    for n in range(2, int(np.max(lengths)) + 1):
        offsets[n] = offsets[n - 1] + d ** (n - 1)
    cols = [offsets[int(n)] + int(c) for n, c in zip(lengths, codes)]
    return dense_values[:, cols]


# -- dense truncated tensor algebra (sigcore.py:297-352, logsig.py:42-72) ----------------
# Flat rows hold levels 1..N in canonical order (no epsilon column); the level
# lists below carry the epsilon coefficient as level 0.


def _levels(row, d, N, eps):
    out, off = [np.array(float(eps))], 0
    for n in range(1, N + 1):
        out.append(np.asarray(row[off:off + d**n], dtype=np.float64).reshape((d,) * n))
        off += d**n
    return out


def _flat(levels, N):
    return np.concatenate([levels[n].reshape(-1) for n in range(1, N + 1)])


def dense_product(a, b, d, N):
    """Chen product of two flat signature batches (chen_concat, sigcore.py:321-334)."""
    return np.stack([_flat(_dense_mul(_levels(x, d, N, 1.0), _levels(y, d, N, 1.0), N), N) for x, y in zip(a, b)])


def dense_inverse(a, d, N):
    """Group inverse sum_k (-x)^k (signature_inverse, sigcore.py:337-352)."""
    rows = []
    for r in a:
        x = _levels(r, d, N, 0.0)
        term, acc = _levels(np.zeros_like(r), d, N, 1.0), _levels(np.zeros_like(r), d, N, 1.0)
        for _ in range(N):
            term = [-t for t in _dense_mul(x, term, N)]
            acc = [u + v for u, v in zip(acc, term)]
        rows.append(_flat(acc, N))
    return np.stack(rows)


def dense_log(a, d, N):
    """log(1 + x) = sum_k (-1)^(k+1) x^k / k of flat signature rows (tensor_log, logsig.py:42-56)."""
    rows = []
    for r in a:
        x = _levels(r, d, N, 0.0)
        power, acc = x, [np.zeros_like(t) for t in x]
        for k in range(1, N + 1):
            acc = [u + (1.0 if k % 2 else -1.0) / k * v for u, v in zip(acc, power)]
            power = _dense_mul(power, x, N)
        rows.append(_flat(acc, N))
    return np.stack(rows)


def dense_exp(a, d, N):
    """exp(x) = sum_k x^k / k! of flat Lie-series rows (tensor_exp, logsig.py:59-72)."""
    rows = []
    for r in a:
        x = _levels(r, d, N, 0.0)
        power, acc, fact = x, [np.zeros_like(t) for t in x], 1.0
        for k in range(1, N + 1):
            fact *= k
            acc = [u + v / fact for u, v in zip(acc, power)]
            power = _dense_mul(power, x, N)
        rows.append(_flat(acc, N))
    return np.stack(rows)


def lyndon_logsig(X, d, N, lyndon_codes, lyndon_lengths):
    """Log-signature at Lyndon words = tensor log of the dense signature restricted to them
    (the identity the reference tests, test_logsig.py:75-87)."""
    full = dense_log(dense_signature(X, d, N), d, N)
    return dense_columns(lyndon_codes, lyndon_lengths, d, full)


def finite_difference_grad(X, codes, lengths, d, upstream, h=1e-5):
    X = np.asarray(X, dtype=np.float64)
    up = np.asarray(upstream, dtype=np.float64)

    def loss(s):
        return np.sum(forward(s, codes, lengths, d) * up, axis=1)

    grads = np.zeros_like(X)
    for j in range(X.shape[1]):
        for i in range(X.shape[2]):
            step = h * np.maximum(1.0, np.abs(X[:, j, i]))
            plus = X.copy()
            plus[:, j, i] += step
            minus = X.copy()
            minus[:, j, i] -= step
            grads[:, j, i] = (loss(plus) - loss(minus)) / (2 * step)
    return grads


def rel_err(actual, expected) -> float:
    """max|a-e| / max(1, max|e|) -- the reference's parity metric (tests/helpers.py:6-11)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    if a.size == 0:
        return 0.0
    scale = max(1.0, float(np.max(np.abs(e))))
    return float(np.max(np.abs(a - e))) / scale
