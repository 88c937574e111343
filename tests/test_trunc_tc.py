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


@pytest.mark.parametrize("L", [2, 5, 9, 33, 100, 257])
def test_tc_forward_matches_oracle(L, monkeypatch):
    ws = sk.build_truncated(16, 4)
    X = brownian(11 + L, 3, L, 16).astype(np.float32)
    out = _forward(X, ws, True, monkeypatch)
    ref = ora.forward(X.astype(np.float64), ws.codes, ws.lengths, 16)
    assert ora.rel_err(out, ref) <= TOL32
    reg = _forward(X, ws, False, monkeypatch)
    assert ora.rel_err(out, reg) <= TOL32


def test_tc_forward_single_sample(monkeypatch):
    ws = sk.build_truncated(16, 4)
    X = np.random.default_rng(0).standard_normal((4, 1, 16)).astype(np.float32)
    out = _forward(X, ws, True, monkeypatch)
    assert out.shape == (4, len(ws)) and not np.any(out)


def test_tc_forward_large_batch_and_include_empty(monkeypatch):
    ws = sk.build_truncated(16, 4, include_empty=True)
    X = brownian(5, 300, 64, 16).astype(np.float32)
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
