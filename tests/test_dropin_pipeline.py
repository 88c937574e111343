"""The numpy drop-in forward streams large results back in chunks (signature._forward_to_host):
the chunked values are bitwise those of one launch, for truncated, fragment and generated-kernel
sets, prefix-closed or not, with and without the epsilon column."""

import importlib

import numpy as np
import pytest
import torch

import paper_2602_24066_b200 as sk
from tests.configs import brownian, build_wordset

pytestmark = pytest.mark.gpu
sigmod = importlib.import_module("paper_2602_24066_b200.signature")  # the module (the package exports a function of that name)


@pytest.mark.parametrize("name", ["c5", "c4", "c3", "non-closed", "eps"])
def test_chunked_numpy_forward_bitwise(name, monkeypatch):
    if name == "non-closed":
        ws = sk.build_custom([(0, 1, 1), (1,), (1, 0, 2), (2, 2, 2, 2), (0, 2), (3, 1, 0)], 4)
    elif name == "eps":
        ws = sk.build_truncated(8, 4, include_empty=True)
    else:
        ws = build_wordset(name, sk)
    B, L = 37, 33
    X = brownian(17, B, L, ws.d).astype(np.float32)
    whole = sk.signature_forward(torch.from_numpy(X).cuda(), ws).values.cpu().numpy()
    monkeypatch.setattr(sigmod, "_PIPE_MIN_BYTES", 1)
    monkeypatch.setattr(sigmod, "_PIPE_CHUNK_BYTES", 5 * ws.width * 4)  # 5-path chunks, ragged tail
    chunked = sk.signature_forward(X, ws).values
    assert isinstance(chunked, np.ndarray)
    assert np.array_equal(chunked, whole)


@pytest.mark.parametrize("name", ["c5", "c4", "c3", "non-closed", "eps"])
@pytest.mark.parametrize("stride", [0, 3])
def test_chunked_numpy_backward_bitwise(name, stride, monkeypatch):
    """gradient._backward_host (upstream staged in chunks through pinned buffers) against one launch
    on device tensors: path and increment gradients bitwise equal."""
    gradmod = importlib.import_module("paper_2602_24066_b200.gradient")
    if name == "non-closed":
        ws = sk.build_custom([(0, 1, 1), (1,), (1, 0, 2), (2, 2, 2, 2), (0, 2), (3, 1, 0)], 4)
    elif name == "eps":
        ws = sk.build_truncated(8, 4, include_empty=True)
    else:
        ws = build_wordset(name, sk)
    B, L = 23, 29
    X = brownian(19, B, L, ws.d)
    g = np.random.default_rng(20).standard_normal((B, ws.width))
    kw = {"checkpoint_stride": stride} if stride else {}
    ref = sk.signature_backward(torch.from_numpy(X).cuda(), ws, torch.from_numpy(g).cuda(), **kw)
    monkeypatch.setattr(gradmod, "_PIPE_MIN_BYTES", 1)
    monkeypatch.setattr(gradmod, "_PIPE_CHUNK_BYTES", 4 * ws.width * 8)  # 4-path chunks, ragged tail
    got = sk.signature_backward(X, ws, g, **kw)
    assert isinstance(got.path_grads, np.ndarray)
    assert np.array_equal(got.path_grads, ref.path_grads.cpu().numpy())
    assert np.array_equal(got.increment_grads, ref.increment_grads.cpu().numpy())
