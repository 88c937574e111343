"""ctypes binding of the C ABI in include/sigkit_b200.h (libsigkit_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2602_24066_b200.build``).  There is no fallback: if the
library or a CUDA device is missing every compute call raises.
"""

from __future__ import annotations

import ctypes
import os

from . import exceptions as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsigkit_b200.so")
# developer override (ablation / A-B builds under tools/); the product path is LIB_PATH
if os.environ.get("SIGB_LIB_PATH"):
    LIB_PATH = os.environ["SIGB_LIB_PATH"]

SIGB_OK = 0
SIGB_F32 = 0
SIGB_F64 = 1

_ERRORS = {
    1: E.ShapeError,
    2: E.DomainError,
    3: E.CapacityError,
    4: E.UnsupportedWordSetError,
}

_P = ctypes.c_void_p
_I = ctypes.c_int64
_C = ctypes.c_int

# name -> (restype, argtypes); mirrors include/sigkit_b200.h
SIGNATURES = {
    "sigb_version": (ctypes.c_int, []),
    "sigb_last_error": (ctypes.c_char_p, []),
    "sigb_device_sm_count": (ctypes.c_int, []),
    "sigb_set_kernel_policy": (_C, [_C]),
    "sigb_set_tensor_cores": (_C, [_C]),
    "sigb_forward_ctas": (_I, [_P, _I]),
    "sigb_launch_count": (ctypes.c_longlong, []),
    "sigb_timing_enable": (_C, [_C]),
    "sigb_timing_read": (_C, [_C, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I)]),
    "sigb_wordset_tables": (_C, [_P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "sigb_plan_create": (_C, [_P, _P, _I, _I, ctypes.POINTER(_P), _P]),
    "sigb_plan_destroy": (_C, [_P]),
    "sigb_plan_closure_size": (_I, [_P]),
    "sigb_plan_num_parts": (_I, [_P]),
    "sigb_plan_step_fmas": (_I, [_P]),
    "sigb_plan_kernel_kind": (_C, [_P]),
    "sigb_fragment_plan_info": (_C, [_P, _P, _I, _I, _P]),
    "sigb_jit_source": (_C, [_P, _P, _I, _I, _C, _C, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "sigb_jit_precompile": (_C, [_P, _P, _I, _I, _C, _C]),
    "sigb_forward": (_C, [_P, _C, _P, _I, _I, _P, _I, _I, _C, _P, _P]),
    "sigb_windows": (_C, [_P, _C, _P, _I, _I, _P, _I, _P, _P]),
    "sigb_backward_workspace_size": (_C, [_P, _C, _I, _I, _I, ctypes.POINTER(ctypes.c_size_t)]),
    "sigb_backward": (_C, [_P, _C, _P, _I, _I, _P, _I, _I, _C, _P, _I, _I, _I, _P, ctypes.c_size_t,
                           _P, _P, _P]),
    "sigb_logsig_forward": (_C, [_C, _P, _I, _I, _P, _P, _P, _I, _C, _P, _I, _P]),
    "sigb_logsig_backward": (_C, [_C, _P, _I, _I, _P, _I, _P, _P, _P, _P, _P, _C, _I, _P, _I, _P]),
    "sigb_tensor_mul": (_C, [_C, _P, _P, _I, _I, _C, ctypes.c_double, ctypes.c_double, _P, _P]),
}

_lib = None


class ExtensionMissing(RuntimeError):
    """The CUDA extension was not built or cannot be loaded."""


def lib():
    """Load libsigkit_b200.so once; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == SIGB_OK:
        return
    msg = lib().sigb_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, RuntimeError)(msg)


def set_kernel_policy(policy: int) -> None:
    """0 auto (truncated > generated > fragment > level), 1 level only, 2 fragment first, 4 generated first."""
    check(lib().sigb_set_kernel_policy(int(policy)))


def set_tensor_cores(on: bool) -> bool:
    """Process-wide: tensor-core kernels for fp32 d=16 depth-4 truncations (default on); see
    include/sigkit_b200.h sigb_set_tensor_cores for the precision contract.  Returns the previous value."""
    return bool(lib().sigb_set_tensor_cores(1 if on else 0))


def launch_count() -> int:
    return int(lib().sigb_launch_count())


def timing_enable(on: bool = True) -> None:
    """Arm (and reset) CUDA-event timing of the main Chen kernels."""
    check(lib().sigb_timing_enable(int(on)))


def timing_read(which: int) -> tuple[float, int]:
    """(device ms, launches) of the forward (0) / backward (1) kernel since the last read."""
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    check(lib().sigb_timing_read(int(which), ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def fragment_plan_info(codes, lengths, d: int) -> dict:
    """Host-only fragment decomposition of a word set (sigb_fragment_plan_info; no device needed)."""
    import numpy as np

    c = np.ascontiguousarray(codes, dtype=np.uint64)
    n = np.ascontiguousarray(lengths, dtype=np.int64)
    info = np.zeros(8, dtype=np.int64)
    check(lib().sigb_fragment_plan_info(c.ctypes.data, n.ctypes.data, int(n.size), int(d), info.ctypes.data))
    keys = ("NC", "G", "K", "fragments", "ctas_per_path", "closure", "cost", "instantiated")
    return dict(zip(keys, (int(v) for v in info)))


def jit_precompile(codes, lengths, d: int, dtype: int = SIGB_F32, backward: bool = False) -> None:
    """Host-only: compile a small word set's generated kernel into the cubin cache (sigb_jit_precompile)."""
    import numpy as np

    c = np.ascontiguousarray(codes, dtype=np.uint64)
    n = np.ascontiguousarray(lengths, dtype=np.int64)
    check(lib().sigb_jit_precompile(c.ctypes.data, n.ctypes.data, int(n.size), int(d), int(dtype), int(backward)))


def jit_source(codes, lengths, d: int, dtype: int = SIGB_F32, backward: bool = False) -> str:
    """Host-only: the CUDA source the plan generates for a small word set (sigb_jit_source)."""
    import numpy as np

    c = np.ascontiguousarray(codes, dtype=np.uint64)
    n = np.ascontiguousarray(lengths, dtype=np.int64)
    size = ctypes.c_size_t()
    check(lib().sigb_jit_source(c.ctypes.data, n.ctypes.data, int(n.size), int(d), int(dtype), int(backward), None, 0,
                                ctypes.byref(size)))
    buf = ctypes.create_string_buffer(size.value + 1)
    check(lib().sigb_jit_source(c.ctypes.data, n.ctypes.data, int(n.size), int(d), int(dtype), int(backward), buf,
                                size.value + 1, ctypes.byref(size)))
    return buf.value.decode()
