"""The C-ABI boundary (include/sigkit_b200.h) without a GPU.

Checks that libsigkit_b200.so loads, exports every function the header
declares, that the ctypes table in _lib.py binds exactly those functions,
and the host-only entry points (no device work).
"""

import ctypes
import os
import re

import pytest

from paper_2602_24066_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sigkit_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sigb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2602_24066_b200 import build

        build.build()
    return ctypes.CDLL(_lib.LIB_PATH)


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ("sigb_wordset_tables", "sigb_plan_create", "sigb_forward", "sigb_windows",
                 "sigb_backward", "sigb_backward_workspace_size", "sigb_last_error"):
        assert must in names


def test_library_exports_every_header_symbol(so):
    missing = [n for n in header_functions() if not hasattr(so, n)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_host_only_entry_points():
    L = _lib.lib()
    assert L.sigb_version() == 100
    # invalid arguments fail with a code and a message, without touching a device
    assert L.sigb_set_kernel_policy(7) == 2
    assert b"policy" in L.sigb_last_error()
    assert L.sigb_set_kernel_policy(3) == 2  # the removed level-slot family
    assert L.sigb_set_kernel_policy(0) == 0
    assert L.sigb_plan_closure_size(None) == -1
    assert L.sigb_forward(None, 0, None, 1, 2, None, 1, 0, 0, None, None) == 2
    ms = ctypes.c_double()
    assert L.sigb_timing_read(5, ctypes.byref(ms), None) == 2
    with pytest.raises(_lib._ERRORS[2]):
        _lib.check(L.sigb_set_kernel_policy(-1))


def test_error_codes_map_to_reference_hierarchy():
    from paper_2602_24066_b200 import exceptions as E

    assert _lib._ERRORS == {1: E.ShapeError, 2: E.DomainError, 3: E.CapacityError,
                            4: E.UnsupportedWordSetError}
    for cls in _lib._ERRORS.values():
        assert issubclass(cls, E.SigkitError)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_fragment_planner_covers_configs(name):
    """The host-only fragment planner cuts every config's closure with full ownership coverage."""
    import paper_2602_24066_b200 as sk
    from tests.configs import build_wordset

    ws = build_wordset(name, sk)
    info = _lib.fragment_plan_info(ws.codes, ws.lengths, ws.d)
    assert info["closure"] == len(ws)  # all five sets are prefix-closed
    assert info["instantiated"] == 1
    assert 1 <= info["NC"] <= 5 and info["fragments"] >= 1
    assert info["ctas_per_path"] == -(-info["fragments"] // 128)


def test_fragment_planner_random_sets():
    import numpy as np

    import paper_2602_24066_b200 as sk

    rng = np.random.default_rng(0)
    for _ in range(40):
        d = int(rng.integers(1, 20))
        words = {tuple(int(x) for x in rng.integers(0, d, int(rng.integers(1, 7)))) for _ in range(50)}
        ws = sk.build_custom(sorted(words), d)
        info = _lib.fragment_plan_info(ws.codes, ws.lengths, ws.d)
        closure = {w[:k] for w in words for k in range(1, len(w) + 1)}
        assert info["closure"] == len(closure)


def test_generated_source_for_small_sets():
    """The code generator (host-only) emits a kernel per direction with one case per task."""
    import paper_2602_24066_b200 as sk
    from tests.configs import build_wordset

    ws = build_wordset("c3", sk)
    fwd = _lib.jit_source(ws.codes, ws.lengths, ws.d, _lib.SIGB_F32, False)
    bwd = _lib.jit_source(ws.codes, ws.lengths, ws.d, _lib.SIGB_F64, True)
    assert 'extern "C" __global__' in fwd and "sigjit_fwd" in fwd and "typedef float R;" in fwd
    assert "sigjit_bwd" in bwd and "typedef double R;" in bwd
    assert fwd.count("case ") >= 2 and bwd.count("case ") >= fwd.count("case ")
    with pytest.raises(_lib._ERRORS[4]):
        big = build_wordset("c4", sk)
        _lib.jit_source(big.codes, big.lengths, big.d, _lib.SIGB_F32, False)
