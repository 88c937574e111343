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
