"""GPU parity: the CUDA path (through the C ABI) against the reference's outputs.

Golden vectors come from the reference package itself (tests/golden/); the C
oracle (oracle/) covers sizes the fixtures do not.  Gates (BASELINE.json
north_star): index tables bit-exact; fp64 within 1e-10 relative; fp32
within 1e-4 relative to the fp64 oracle -- metric rel_err = max|a-e| /
max(1, max|e|) (reference tests/helpers.py:6-11).
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2602_24066_b200 as sk
from oracle import oracle as ora
from tests.configs import CONFIGS, brownian, build_wordset

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4
SMALL_SETS = ("trunc_3_3", "trunc_2_4_eps", "trunc_1_3", "aniso_12_4", "aniso_123_5",
              "custom_np1", "custom_np2", "custom_missing", "c3")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def ws_from_golden(t, key):
    d = int(t[f"{key}/d"])
    return sk.WordSet(d, t[f"{key}/lengths"], t[f"{key}/codes"], include_empty=bool(t[f"{key}/include_empty"]))


# -- (1) word-set tables on device: bit-exact -----------------------------------------------


@pytest.mark.parametrize("key", SMALL_SETS)
def test_device_tables_bit_exact(golden_tables, key):
    ws = ws_from_golden(golden_tables, key)
    assert np.array_equal(ws.letters, golden_tables[f"{key}/letters"])
    assert np.array_equal(ws.prefix_table, golden_tables[f"{key}/prefix"])
    assert np.array_equal(ws.suffix_table, golden_tables[f"{key}/suffix"])
    lo = ws.level_offsets
    for n in range(1, ws.max_len + 1):
        s = ws.level_slice(n)
        assert (lo[n], lo[n + 1]) == (s.start, s.stop)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_device_tables_configs_bit_exact(golden_meta, name):
    m = golden_meta["wordsets"][name]
    ws = build_wordset(name, sk)
    assert len(ws) == m["W"] and ws.max_len == m["max_len"]
    assert sha(ws.codes) == m["codes_sha"] and sha(ws.lengths) == m["lengths_sha"]
    assert sha(ws.letters) == m["letters_sha"]
    assert sha(ws.prefix_table) == m["prefix_sha"]
    assert sha(ws.suffix_table) == m["suffix_sha"]
    assert ws.is_full_truncation == m["is_full_truncation"]


def test_packed_letters_match_pack_letters():
    from paper_2602_24066_b200.device import wordset_tables

    ws = sk.build_anisotropic(sk.AnisotropyWeights((1.0, 2.0, 3.0), 5.0))
    packed = wordset_tables(ws.codes, ws.lengths, ws.d)["packed"]
    b = sk.Alphabet(ws.d).bits_per_letter
    for i, w in enumerate(ws.words):
        assert int(packed[i]) == sk.pack_letters(w, b, ws.d).bits


# -- (2) forward ----------------------------------------------------------------------------------


def test_forward_kats(golden_forward):
    g = golden_forward
    ws = sk.build_truncated(2, 2)
    for key in ("kat_segment", "kat_lpath"):
        out = sk.signature_forward(g[f"{key}/X"], ws).values
        np.testing.assert_allclose(out, g[f"{key}/S"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(sk.signature_forward(g["kat_lpath/X"], ws).values[0],
                               [1.0, 1.0, 0.5, 1.0, 0.0, 0.5], atol=1e-15)


def test_forward_constant_and_single_sample():
    assert np.all(sk.signature_forward(np.zeros((2, 6, 3)), sk.build_truncated(3, 3)).values == 0.0)
    assert np.all(sk.signature_forward(np.ones((1, 1, 2)), sk.build_truncated(2, 3)).values == 0.0)


def test_forward_include_empty():
    ws = sk.build_truncated(2, 1, include_empty=True)
    out = sk.signature_forward(np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]]), ws)
    assert out.values.shape == (1, 3) and out.values[0, 0] == 1.0
    assert out.column_names() == ["e", "1", "2"]


def test_forward_empty_batch():
    out = sk.signature_forward(np.zeros((0, 5, 2)), sk.build_truncated(2, 2))
    assert out.values.shape == (0, 6)


def test_forward_small_cases(golden_forward):
    g = golden_forward
    for i, (d, N) in enumerate(g["small/dN"]):
        out = sk.signature_forward(g[f"small{i}/X"], sk.build_truncated(int(d), int(N))).values
        assert ora.rel_err(out, g[f"small{i}/S"]) <= 1e-12, i


@pytest.mark.parametrize("key", ["custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"])
def test_forward_sets(golden_forward, golden_tables, key):
    g = golden_forward
    ws = ws_from_golden(golden_tables, key)
    assert ora.rel_err(sk.signature_forward(g[f"{key}/X"], ws).values, g[f"{key}/S"]) <= 1e-12
    out32 = sk.signature_forward(g[f"{key}/X32"], ws).values
    assert out32.dtype == np.float32
    assert ora.rel_err(out32, g[f"{key}/S"]) <= 1e-5


@pytest.mark.parametrize("name", list(CONFIGS))
def test_forward_config_subsets(golden_forward, name):
    g = golden_forward
    ws = build_wordset(name, sk)
    out = sk.signature_forward(g[f"{name}/X"], ws).values
    tol = TOL64 if CONFIGS[name]["dtype"] == np.float64 else TOL32
    assert ora.rel_err(out, g[f"{name}/S64"]) <= tol


def test_forward_c1_full_config():
    cfg = CONFIGS["c1"]
    ws = build_wordset("c1", sk)
    X = brownian(cfg["seed"], cfg["B"], cfg["L"], cfg["d"])
    out = sk.signature_forward(X, ws).values
    np.testing.assert_allclose(out[0, :4], [-0.15336914440166166, 0.22210567119876828,
                                            -1.7218293032451484, -0.10731244354544103], rtol=1e-10)
    assert ora.rel_err(out, ora.forward(X, ws.codes, ws.lengths, 4)) <= TOL64


def test_forward_reparametrisation_bitwise():
    rng = np.random.default_rng(44)
    base = rng.random((2, 6, 3)) * 2 - 1
    dup = np.concatenate([base[:, :3], base[:, 2:]], axis=1)
    ws = sk.build_truncated(3, 3)
    assert np.array_equal(sk.signature_forward(base, ws).values, sk.signature_forward(dup, ws).values)


def test_forward_deterministic_bitwise():
    X = brownian(5, 64, 65, 16).astype(np.float32)
    ws = build_wordset("c5", sk)
    a = sk.signature_forward(X, ws).values
    b = sk.signature_forward(X, ws).values
    assert np.array_equal(a, b)


def test_windows(golden_forward):
    g = golden_forward
    outs = sk.signature_windows(g["windows/X"], sk.build_truncated(2, 3), sk.WindowSpec(g["windows/pairs"]))
    for k, o in enumerate(outs):
        assert ora.rel_err(o.values, g["windows/S"][:, k]) <= 1e-12
    with pytest.raises(sk.WindowError):
        sk.signature_windows(np.zeros((1, 4, 2)), sk.build_truncated(2, 2), sk.WindowSpec(np.array([[0, 5]])))


def test_shape_errors():
    with pytest.raises(sk.ShapeError, match="word set has d=2 but paths have 3 channels"):
        sk.signature_forward(np.zeros((1, 3, 3)), sk.build_truncated(2, 2))
    x = np.zeros((1, 2, 1))
    x[0, 1, 0] = np.nan
    with pytest.raises(sk.DomainError):
        sk.signature_forward(x, sk.build_truncated(1, 2))


# -- (3) backward ------------------------------------------------------------------------------------


def test_backward_small_cases(golden_backward):
    g = golden_backward
    for i, (d, N) in enumerate(g["small/dN"]):
        out = sk.signature_backward(g[f"small{i}/X"], sk.build_truncated(int(d), int(N)), g[f"small{i}/g"])
        assert out.path_grads.dtype == np.float64
        assert ora.rel_err(out.path_grads, g[f"small{i}/dX"]) <= TOL64, i
        assert ora.rel_err(out.increment_grads, g[f"small{i}/dInc"]) <= TOL64, i


@pytest.mark.parametrize("key", ["custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"])
def test_backward_sets(golden_backward, golden_tables, key):
    g = golden_backward
    ws = ws_from_golden(golden_tables, key)
    dX = sk.signature_backward(g[f"{key}/X"], ws, g[f"{key}/g"]).path_grads
    assert ora.rel_err(dX, g[f"{key}/dX"]) <= TOL64
    fd = g[f"{key}/dX_fd"]
    assert np.max(np.abs(dX - fd) / np.maximum(1.0, np.maximum(np.abs(dX), np.abs(fd)))) <= 1e-6


def test_backward_checkpoint_stride(golden_backward):
    g = golden_backward
    ws = sk.build_truncated(2, 3)
    plain = sk.signature_backward(g["ckpt/X"], ws, g["ckpt/g"]).path_grads
    ck = sk.signature_backward(g["ckpt/X"], ws, g["ckpt/g"], checkpoint_stride=5).path_grads
    assert ora.rel_err(plain, g["ckpt/dX_plain"]) <= TOL64
    assert ora.rel_err(ck, g["ckpt/dX_c5"]) <= TOL64
    assert ora.rel_err(ck, plain) <= 1e-9


@pytest.mark.parametrize("name", list(CONFIGS))
def test_backward_config_subsets_fp64(golden_backward, name):
    g = golden_backward
    ws = build_wordset(name, sk)
    dX = sk.signature_backward(g[f"{name}/X"], ws, g[f"{name}/g"]).path_grads
    assert ora.rel_err(dX, g[f"{name}/dX"]) <= TOL64


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_autograd_fp32_config_subsets(golden_backward, name):
    g = golden_backward
    ws = build_wordset(name, sk)
    X = torch.from_numpy(g[f"{name}/X"].astype(np.float32)).cuda().requires_grad_(True)
    S = sk.signature(X, ws)
    assert S.dtype == torch.float32
    S.backward(torch.from_numpy(g[f"{name}/g"]).float().cuda())
    assert ora.rel_err(X.grad.cpu().numpy(), g[f"{name}/dX"]) <= TOL32


def test_backward_level_one_closed_form():
    rng = np.random.default_rng(3)
    X = rng.random((2, 6, 3)) * 2 - 1
    ws = sk.build_truncated(3, 1)
    gr = rng.normal(size=(2, 3))
    out = sk.signature_backward(X, ws, gr).path_grads
    np.testing.assert_allclose(out[:, 0], -gr, atol=1e-15)
    np.testing.assert_allclose(out[:, -1], gr, atol=1e-15)
    assert np.all(out[:, 1:-1] == 0.0)


def test_backward_zero_upstream_linearity_sum_zero():
    rng = np.random.default_rng(7)
    X = rng.random((2, 6, 2)) * 2 - 1
    ws = sk.build_truncated(2, 3)
    assert np.all(sk.signature_backward(X, ws, np.zeros((2, len(ws)))).path_grads == 0.0)
    g1, g2 = rng.normal(size=(2, len(ws))), rng.normal(size=(2, len(ws)))
    comb = sk.signature_backward(X, ws, 1.7 * g1 + g2).path_grads
    sep = 1.7 * sk.signature_backward(X, ws, g1).path_grads + sk.signature_backward(X, ws, g2).path_grads
    assert ora.rel_err(comb, sep) <= 1e-12
    np.testing.assert_allclose(sk.signature_backward(X, ws, g1).path_grads.sum(axis=1), 0.0, atol=1e-12)


def test_backward_eps_column_and_upcast():
    rng = np.random.default_rng(11)
    X = rng.random((1, 5, 2)) * 2 - 1
    ws = sk.build_truncated(2, 2, include_empty=True)
    gr = rng.normal(size=(1, len(ws)))
    a = sk.signature_backward(X, ws, gr).path_grads
    b = sk.signature_backward(X, ws, np.concatenate([np.ones((1, 1)), gr], axis=1)).path_grads
    assert np.array_equal(a, b)
    c = sk.signature_backward(X.astype(np.float32), ws, gr).path_grads
    assert c.dtype == np.float64 and ora.rel_err(a, c) <= 1e-6


def test_backward_single_sample_and_errors():
    ws = sk.build_truncated(2, 2)
    out = sk.signature_backward(np.ones((2, 1, 2)), ws, np.ones((2, len(ws))))
    assert out.path_grads.shape == (2, 1, 2) and np.all(out.path_grads == 0)
    with pytest.raises(sk.ShapeError):
        sk.signature_backward(np.zeros((1, 3, 2)), ws, np.zeros((2, len(ws))))
    with pytest.raises(sk.ShapeError):
        sk.signature_backward(np.zeros((1, 3, 2)), ws, np.zeros((1, 3)))
    with pytest.raises(sk.DomainError):
        sk.signature_backward(np.zeros((1, 3, 2)), ws, np.zeros((1, len(ws))), checkpoint_stride=0)


def test_backward_deterministic_bitwise():
    X = brownian(4, 8, 65, 10)
    ws = build_wordset("c4", sk)
    g = np.random.default_rng(0).standard_normal((8, len(ws)))
    a = sk.signature_backward(X, ws, g).path_grads
    b = sk.signature_backward(X, ws, g).path_grads
    assert np.array_equal(a, b)


def test_autograd_gradcheck_fp64():
    ws = sk.build_custom([(1, 0), (0, 1, 1), (1, 1, 0, 0)], 2)
    X = torch.rand(2, 6, 2, dtype=torch.float64, device="cuda", requires_grad=True)
    assert torch.autograd.gradcheck(lambda x: sk.signature(x, ws), (X,), eps=1e-6, atol=1e-7)


def test_module_wrapper():
    ws = sk.build_truncated(3, 3, include_empty=True)
    m = sk.Signature(ws)
    X = torch.rand(4, 9, 3, dtype=torch.float64, device="cuda", requires_grad=True)
    S = m(X)
    assert S.shape == (4, len(ws) + 1) and bool((S[:, 0] == 1).all())
    S.sum().backward()
    gr = np.ones((4, len(ws) + 1))
    ref = sk.signature_backward(X.detach().cpu().numpy(), ws, gr).path_grads
    assert ora.rel_err(X.grad.cpu().numpy(), ref) <= 1e-12


# -- both kernel families on the truncated configs ------------------------------------------------


@pytest.fixture(params=[0, 1], ids=["auto", "generic"])
def policy(request):
    from paper_2602_24066_b200 import _lib

    _lib.set_kernel_policy(request.param)
    yield request.param
    _lib.set_kernel_policy(0)


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_truncated_paths_both_kernels(golden_forward, golden_backward, policy, name):
    ws = build_wordset(name, sk)
    g = golden_forward
    out = sk.signature_forward(g[f"{name}/X"], ws).values
    tol = TOL64 if CONFIGS[name]["dtype"] == np.float64 else TOL32
    assert ora.rel_err(out, g[f"{name}/S64"]) <= tol
    gb = golden_backward
    dX = sk.signature_backward(gb[f"{name}/X"], ws, gb[f"{name}/g"]).path_grads
    assert ora.rel_err(dX, gb[f"{name}/dX"]) <= TOL64
    X = torch.from_numpy(gb[f"{name}/X"].astype(np.float32)).cuda().requires_grad_(True)
    sk.signature(X, ws).backward(torch.from_numpy(gb[f"{name}/g"]).float().cuda())
    assert ora.rel_err(X.grad.cpu().numpy(), gb[f"{name}/dX"]) <= TOL32


@pytest.mark.parametrize("d,N", [(4, 4), (4, 5), (4, 6), (8, 4), (8, 5), (16, 3), (16, 4)])
def test_truncated_instantiations_vs_oracle(d, N):
    ws = sk.build_truncated(d, N, include_empty=True)
    rng = np.random.default_rng(d * 10 + N)
    B = 5
    X = brownian(d + N, B, 9, d)
    out = sk.signature_forward(X, ws).values
    assert out[:, 0].tolist() == [1.0] * B
    ref = ora.forward(X, ws.codes, ws.lengths, d)
    assert ora.rel_err(out[:, 1:], ref) <= TOL64
    g = rng.standard_normal((B, len(ws) + 1))
    dX = sk.signature_backward(X, ws, g).path_grads
    _, dref = ora.backward(X, ws.codes, ws.lengths, d, g[:, 1:])
    assert ora.rel_err(dX, dref) <= TOL64
    X32 = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
    S32 = sk.signature(X32, ws)
    S32.backward(torch.from_numpy(g).float().cuda())
    assert ora.rel_err(S32.detach().cpu().numpy()[:, 1:], ref) <= TOL32
    assert ora.rel_err(X32.grad.cpu().numpy(), dref) <= TOL32


def test_truncated_batch_tails():
    # batch sizes that do not fill the paths-per-CTA tiling of the d=4 kernel
    ws = sk.build_truncated(4, 4)
    for B in (1, 3, 17, 33):
        X = brownian(B, B, 20, 4)
        g = np.random.default_rng(B).standard_normal((B, len(ws)))
        assert ora.rel_err(sk.signature_forward(X, ws).values, ora.forward(X, ws.codes, ws.lengths, 4)) <= TOL64
        _, dref = ora.backward(X, ws.codes, ws.lengths, 4, g)
        assert ora.rel_err(sk.signature_backward(X, ws, g).path_grads, dref) <= TOL64
