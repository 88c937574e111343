"""Pin the C oracle (oracle/sig_oracle.c) against the reference's own outputs.

The golden vectors were produced by importing the reference package
(tests/golden/make_golden.py).  CPU only.
"""

import numpy as np
import pytest

from oracle import oracle as ora

SMALL_SETS = ("trunc_3_3", "trunc_2_4_eps", "trunc_1_3", "aniso_12_4", "aniso_123_5",
              "custom_np1", "custom_np2", "custom_missing", "c3")


@pytest.mark.parametrize("key", SMALL_SETS)
def test_tables_bit_exact(golden_tables, key):
    g = golden_tables
    codes, lengths, d = g[f"{key}/codes"], g[f"{key}/lengths"], int(g[f"{key}/d"])
    assert np.array_equal(ora.letters(codes, lengths, d), g[f"{key}/letters"])
    assert np.array_equal(ora.factor_table(codes, lengths, d, False), g[f"{key}/prefix"])
    assert np.array_equal(ora.factor_table(codes, lengths, d, True), g[f"{key}/suffix"])


def _trunc(d, N):
    lengths = np.concatenate([np.full(d**n, n, dtype=np.int64) for n in range(1, N + 1)])
    codes = np.concatenate([np.arange(d**n, dtype=np.uint64) for n in range(1, N + 1)])
    return codes, lengths


def test_forward_kats(golden_forward):
    g = golden_forward
    codes, lengths = _trunc(2, 2)
    for key in ("kat_segment", "kat_lpath"):
        assert np.array_equal(ora.forward(g[f"{key}/X"], codes, lengths, 2), g[f"{key}/S"])
    np.testing.assert_allclose(g["kat_segment/S"][0], [1.0, 2.0, 0.5, 1.0, 1.0, 2.0], rtol=1e-15)


def test_forward_small_bitwise(golden_forward):
    g = golden_forward
    for i, (d, N) in enumerate(g["small/dN"]):
        codes, lengths = _trunc(int(d), int(N))
        X = g[f"small{i}/X"]
        ours = ora.forward(X, codes, lengths, int(d))
        assert np.array_equal(ours, g[f"small{i}/S"]), i
        assert ora.rel_err(ours, ora.dense_signature(X, int(d), int(N))) <= 1e-12


@pytest.mark.parametrize("key", ["custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"])
def test_forward_sets_bitwise(golden_forward, golden_tables, key):
    g, t = golden_forward, golden_tables
    codes, lengths, d = t[f"{key}/codes"], t[f"{key}/lengths"], int(t[f"{key}/d"])
    assert np.array_equal(ora.forward(g[f"{key}/X"], codes, lengths, d), g[f"{key}/S"])
    assert np.array_equal(ora.forward(g[f"{key}/X32"], codes, lengths, d), g[f"{key}/S32"])


def test_forward_c1_and_c3_bitwise(golden_forward, golden_tables):
    g, t = golden_forward, golden_tables
    codes, lengths = _trunc(4, 4)
    assert np.array_equal(ora.forward(g["c1/X"], codes, lengths, 4), g["c1/S"])
    codes, lengths = t["c3/codes"], t["c3/lengths"]
    assert np.array_equal(ora.forward(g["c3/X"], codes, lengths, 16), g["c3/S"])


def test_windows_bitwise(golden_forward):
    g = golden_forward
    codes, lengths = _trunc(2, 3)
    ours = ora.windows(g["windows/X"], codes, lengths, 2, g["windows/pairs"])
    assert np.array_equal(ours, g["windows/S"])


def test_backward_small_bitwise(golden_backward):
    g = golden_backward
    for i, (d, N) in enumerate(g["small/dN"]):
        codes, lengths = _trunc(int(d), int(N))
        ig, pg = ora.backward(g[f"small{i}/X"], codes, lengths, int(d), g[f"small{i}/g"])
        assert np.array_equal(pg, g[f"small{i}/dX"]), i
        assert np.array_equal(ig, g[f"small{i}/dInc"]), i


@pytest.mark.parametrize("key", ["custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"])
def test_backward_sets(golden_backward, golden_tables, key):
    g, t = golden_backward, golden_tables
    codes, lengths, d = t[f"{key}/codes"], t[f"{key}/lengths"], int(t[f"{key}/d"])
    _, pg = ora.backward(g[f"{key}/X"], codes, lengths, d, g[f"{key}/g"])
    assert np.array_equal(pg, g[f"{key}/dX"])


def test_backward_checkpoint(golden_backward):
    g = golden_backward
    codes, lengths = _trunc(2, 3)
    _, plain = ora.backward(g["ckpt/X"], codes, lengths, 2, g["ckpt/g"])
    _, ck = ora.backward(g["ckpt/X"], codes, lengths, 2, g["ckpt/g"], stride=5)
    assert np.array_equal(plain, g["ckpt/dX_plain"])
    assert np.array_equal(ck, g["ckpt/dX_c5"])


def test_backward_c1_bitwise(golden_backward):
    g = golden_backward
    codes, lengths = _trunc(4, 4)
    _, pg = ora.backward(g["c1/X"], codes, lengths, 4, g["c1/g"])
    assert np.array_equal(pg, g["c1/dX"])


def test_thread_count_invariance():
    rng = np.random.default_rng(9)
    X = rng.random((3, 7, 2))
    codes, lengths = _trunc(2, 3)
    g = rng.normal(size=(3, len(codes)))
    ora.set_threads(1)
    a = ora.forward(X, codes, lengths, 2), ora.backward(X, codes, lengths, 2, g)[1]
    ora.set_threads(4)
    b = ora.forward(X, codes, lengths, 2), ora.backward(X, codes, lengths, 2, g)[1]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
