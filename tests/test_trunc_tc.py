"""Tensor-core truncated forward (csrc/sigb_trunc_tc.cuh, SIGB_TRUNC_TC=1) against
the fp64 oracle and the register kernel: fp32 gate 1e-4 (north_star), the
reference's rel_err metric (tests/helpers.py:6-11)."""

import numpy as np
import pytest
import torch

import paper_2602_24066_b200 as sk
from oracle import oracle as ora
from tests.configs import brownian

pytestmark = pytest.mark.gpu

TOL32 = 1e-4


def _forward(X, ws, tc, monkeypatch):
    monkeypatch.setenv("SIGB_TRUNC_TC", "1" if tc else "0")
    return sk.signature_forward(X, ws).values


@pytest.mark.parametrize("d,N", [(16, 4)])
@pytest.mark.parametrize("L", [2, 5, 9, 33, 100, 257])
def test_tc_forward_matches_oracle(d, N, L, monkeypatch):
    ws = sk.build_truncated(d, N)
    X = brownian(11 + L, 3, L, d).astype(np.float32)
    out = _forward(X, ws, True, monkeypatch)
    ref = ora.forward(X.astype(np.float64), ws.codes, ws.lengths, d)
    assert ora.rel_err(out, ref) <= TOL32
    reg = _forward(X, ws, False, monkeypatch)
    assert ora.rel_err(out, reg) <= TOL32


def test_tc_forward_single_sample(monkeypatch):
    ws = sk.build_truncated(16, 4)
    X = np.random.default_rng(0).standard_normal((4, 1, 16)).astype(np.float32)
    out = _forward(X, ws, True, monkeypatch)
    assert out.shape == (4, len(ws)) and not np.any(out)


@pytest.mark.parametrize("d,N", [(16, 4)])
def test_tc_forward_large_batch_and_include_empty(d, N, monkeypatch):
    ws = sk.build_truncated(d, N, include_empty=True)
    X = brownian(5, 300, 64, d).astype(np.float32)
    out = _forward(X, ws, True, monkeypatch)
    reg = _forward(X, ws, False, monkeypatch)
    assert np.all(out[:, 0] == 1.0)
    assert ora.rel_err(out, reg) <= TOL32


def test_tc_forward_deterministic(monkeypatch):
    ws = sk.build_truncated(16, 4)
    X = torch.randn(64, 129, 16, device="cuda").cumsum(1) * 0.1
    monkeypatch.setenv("SIGB_TRUNC_TC", "1")
    a = sk.signature(X, ws)
    b = sk.signature(X, ws)
    assert torch.equal(a, b)


# -- backward on the tensor cores: SIGB_TRUNC_TC_BWD = "2" the P/Q kernel (sigb_trunc_pq.cuh, the
# default), "1" the intermediate kernel with only tb = Lambda . dX on tcgen05 (TcBwd, sigb_trunc.cuh;
# d = 16 only -- d = 8 falls back to the CUDA cores), "0" the CUDA-core kernel ------------------------

BWD_MODES = ["2", "1"]


def _autograd(X, ws, g, mode, monkeypatch):
    monkeypatch.setenv("SIGB_TRUNC_TC_BWD", mode)
    Xt = torch.from_numpy(X).cuda().requires_grad_(True)
    S = sk.signature(Xt, ws)
    S.backward(torch.from_numpy(g).cuda())
    return Xt.grad.cpu().numpy()


@pytest.mark.parametrize("mode", BWD_MODES)
@pytest.mark.parametrize("d,N", [(16, 4), (8, 5)])
@pytest.mark.parametrize("L", [2, 3, 17, 18, 33, 34, 49, 65, 200])
def test_tc_backward_matches_oracle(d, N, L, mode, monkeypatch):
    """Chunk and MMA-group edges (M = 1, M < 16, M = 16 / 17 (second group empty / one step), M = 32,
    M = 33, M = 48, ragged last chunk) against the fp64 oracle and the CUDA-core backward, for both
    P/Q instantiations (config 5 and config 2 sets)."""
    ws = sk.build_truncated(d, N)
    B = 3
    X = brownian(40 + L, B, L, d).astype(np.float32)
    g = np.random.default_rng(L).standard_normal((B, len(ws))).astype(np.float32)
    dX = _autograd(X, ws, g, mode, monkeypatch)
    _, dref = ora.backward(X.astype(np.float64), ws.codes, ws.lengths, d, g.astype(np.float64))
    assert ora.rel_err(dX, dref) <= TOL32
    assert ora.rel_err(dX, _autograd(X, ws, g, "0", monkeypatch)) <= TOL32


@pytest.mark.parametrize("mode", BWD_MODES)
@pytest.mark.parametrize("d,N", [(16, 4), (8, 5)])
def test_tc_backward_scaled_inputs(d, N, mode, monkeypatch):
    """Power-of-two operand scaling: upstream rows spanning 2^-30..2^30, a path scaled by 1e4,
    one by 1e-4, a constant stretch (zero increments), a zero upstream path."""
    ws = sk.build_truncated(d, N)
    B, L = 5, 70
    X = brownian(77, B, L, d)
    X[1] *= 1e4
    X[2] *= 1e-4
    X[3, 20:40] = X[3, 20]
    X = X.astype(np.float32)
    rng = np.random.default_rng(78)
    g = rng.standard_normal((B, len(ws)))
    g *= np.exp2(rng.integers(-30, 31, size=(B, len(ws))))
    g[4] = 0.0
    g = g.astype(np.float32)
    dX = _autograd(X, ws, g, mode, monkeypatch)
    _, dref = ora.backward(X.astype(np.float64), ws.codes, ws.lengths, d, g.astype(np.float64))
    for b in range(B):
        assert ora.rel_err(dX[b], dref[b]) <= TOL32, b
    assert not np.any(dX[4])


@pytest.mark.parametrize("mode", BWD_MODES)
def test_tc_backward_deterministic(mode, monkeypatch):
    ws = sk.build_truncated(16, 4)
    X = brownian(81, 9, 100, 16).astype(np.float32)
    g = np.random.default_rng(82).standard_normal((9, len(ws))).astype(np.float32)
    a = _autograd(X, ws, g, mode, monkeypatch)
    b = _autograd(X, ws, g, mode, monkeypatch)
    assert np.array_equal(a, b)


def test_tensor_core_switch(monkeypatch):
    """sigb_set_tensor_cores (include/sigkit_b200.h): off selects the CUDA-core fp32 kernels for the
    c5-shaped set -- bitwise the SIGB_TRUNC_TC=0 / SIGB_TRUNC_TC_BWD=0 kernels -- on the tensor-core
    ones; both inside the fp32 gate against the fp64 oracle."""
    from paper_2602_24066_b200 import _lib

    ws = sk.build_truncated(16, 4)
    X = brownian(91, 4, 50, 16).astype(np.float32)
    g = np.random.default_rng(92).standard_normal((4, len(ws))).astype(np.float32)
    ref = ora.forward(X.astype(np.float64), ws.codes, ws.lengths, 16)
    _, dref = ora.backward(X.astype(np.float64), ws.codes, ws.lengths, 16, g.astype(np.float64))

    def run():
        Xt = torch.from_numpy(X).cuda().requires_grad_(True)
        S = sk.signature(Xt, ws)
        S.backward(torch.from_numpy(g).cuda())
        return S.detach().cpu().numpy(), Xt.grad.cpu().numpy()

    prev = _lib.set_tensor_cores(False)
    try:
        S_cc, d_cc = run()
    finally:
        _lib.set_tensor_cores(prev)
    S_tc, d_tc = run()
    monkeypatch.setenv("SIGB_TRUNC_TC", "0")
    monkeypatch.setenv("SIGB_TRUNC_TC_BWD", "0")
    S_env, d_env = run()
    assert np.array_equal(S_cc, S_env) and np.array_equal(d_cc, d_env)
    for S, dX in ((S_cc, d_cc), (S_tc, d_tc)):
        assert ora.rel_err(S, ref) <= TOL32
        assert ora.rel_err(dX, dref) <= TOL32


@pytest.mark.parametrize("mode", BWD_MODES)
@pytest.mark.parametrize("d,N", [(16, 4), (8, 5)])
def test_tc_backward_epsilon_column(d, N, mode, monkeypatch):
    """include_empty: the upstream carries a leading epsilon column (g_col0 = 1), so the staged leaf
    block is not 16-byte aligned and the kernel takes its 4-byte copies."""
    ws = sk.build_truncated(d, N, include_empty=True)
    X = brownian(95, 3, 41, d).astype(np.float32)
    g = np.random.default_rng(96).standard_normal((3, len(ws) + 1)).astype(np.float32)
    dX = _autograd(X, ws, g, mode, monkeypatch)
    _, dref = ora.backward(X.astype(np.float64), ws.codes, ws.lengths, d, g[:, 1:].astype(np.float64))
    assert ora.rel_err(dX, dref) <= TOL32
