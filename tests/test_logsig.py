"""Log-signatures and the dense truncated tensor algebra.

Golden vectors come from the reference itself (tests/golden/make_golden_logsig.py:
sigkit.logsignature_forward / _backward, tensor_log / tensor_exp, chen_concat,
signature_inverse).  CPU tests pin the dense oracle and the host-side term
tables against them; GPU tests run the CUDA path (sigb_forward + sigb_logsig_*,
sigb_tensor_mul, sigb_backward) against the same vectors and the reference's
own known answers (/root/reference/pkg/tests/test_logsig.py).
"""

import os

import numpy as np
import pytest

import paper_2602_24066_b200 as sk
from oracle import oracle as ora

HERE = os.path.dirname(os.path.abspath(__file__))
TAGS = ["d1N3", "d2N2", "d2N4", "d3N3", "d4N4", "d3N5"]
L_PATH = np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]])


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(HERE, "golden", "logsig.npz"))


def dN(tag):
    return int(tag[1]), int(tag[3])


# -- CPU: oracle and host tables -----------------------------------------------------------


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_matches_reference(golden, tag):
    d, N = dN(tag)
    g = golden
    X, S = g[f"{tag}_X"], g[f"{tag}_sig"]
    ls = ora.lyndon_logsig(X, d, N, g[f"{tag}_lyndon_codes"], g[f"{tag}_lyndon_lengths"])
    assert ora.rel_err(ls, g[f"{tag}_logsig"]) <= 1e-13
    assert ora.rel_err(ora.dense_log(S, d, N), g[f"{tag}_tlog"]) <= 1e-13
    assert ora.rel_err(ora.dense_exp(ora.dense_log(S, d, N), d, N), g[f"{tag}_texp"]) <= 1e-13
    S2 = ora.dense_signature(g[f"{tag}_Y"], d, N)
    assert ora.rel_err(ora.dense_product(S, S2, d, N), g[f"{tag}_chen"]) <= 1e-13
    assert ora.rel_err(ora.dense_inverse(S, d, N), g[f"{tag}_inv"]) <= 1e-13


@pytest.mark.parametrize("tag", TAGS)
def test_projection_tables_match_reference(golden, tag):
    from paper_2602_24066_b200.logsig import _projection

    d, N = dN(tag)
    pr = _projection(d, N)
    assert np.array_equal(pr.lyndon.codes, golden[f"{tag}_lyndon_codes"])
    assert np.array_equal(pr.lyndon.lengths, golden[f"{tag}_lyndon_lengths"])
    assert np.array_equal(pr.compute.codes, golden[f"{tag}_compute_codes"])
    assert np.array_equal(pr.compute.lengths, golden[f"{tag}_compute_lengths"])
    assert np.array_equal(np.diff(pr.term_off), golden[f"{tag}_nterms"])
    # every column's gradient entries point back at a factor equal to that column
    for c in range(len(pr.compute)):
        for e in pr.entries[pr.col_off[c]:pr.col_off[c + 1]]:
            assert pr.cols[e >> 8, e & 0xFF] == c


def test_width_91_for_d6_n3():
    from paper_2602_24066_b200.logsig import _projection

    assert len(_projection(6, 3).lyndon) == 91


# -- GPU: the CUDA path -------------------------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_logsig_forward_backward_golden(golden, tag):
    d, N = dN(tag)
    X, g = golden[f"{tag}_X"], golden[f"{tag}_g"]
    out = sk.logsignature_forward(X, d, N)
    assert isinstance(out, sk.LogCoefficientBatch)
    assert ora.rel_err(out.values, golden[f"{tag}_logsig"]) <= 1e-12
    gb = sk.logsignature_backward(X, d, N, g)
    assert ora.rel_err(gb.path_grads, golden[f"{tag}_dX"]) <= 1e-10
    # fp32 forward against the fp64 reference on the same (rounded) samples
    out32 = sk.logsignature_forward(X.astype(np.float32), d, N)
    assert out32.values.dtype == np.float32
    assert ora.rel_err(out32.values, golden[f"{tag}_logsig"]) <= 1e-4 * 10


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_tensor_algebra_golden(golden, tag):
    d, N = dN(tag)
    ws = sk.build_truncated(d, N)
    S = sk.signature_forward(golden[f"{tag}_X"], ws)
    S2 = sk.signature_forward(golden[f"{tag}_Y"], ws)
    assert ora.rel_err(S.values, golden[f"{tag}_sig"]) <= 1e-12
    assert ora.rel_err(sk.tensor_log(S).values, golden[f"{tag}_tlog"]) <= 1e-12
    assert ora.rel_err(sk.tensor_exp(sk.tensor_log(S)).values, golden[f"{tag}_texp"]) <= 1e-12
    assert ora.rel_err(sk.chen_concat(S, S2).values, golden[f"{tag}_chen"]) <= 1e-12
    assert ora.rel_err(sk.signature_inverse(S).values, golden[f"{tag}_inv"]) <= 1e-12
    ident = sk.chen_concat(S, sk.signature_inverse(S)).values
    assert np.max(np.abs(ident)) <= 1e-12


@pytest.mark.gpu
def test_reference_known_answers():
    # test_logsig.py:20-27 one-segment log is the increment
    ws = sk.build_truncated(3, 4)
    delta = np.array([0.4, -0.9, 0.2])
    seg = np.stack([np.zeros((1, 3)), delta[None, :]], axis=1)
    log = sk.tensor_log(sk.signature_forward(seg, ws))
    np.testing.assert_allclose(log.values[0, :3], delta, atol=1e-14)
    assert np.max(np.abs(log.values[0, 3:])) <= 1e-14
    # test_logsig.py:35-41 L path
    log = sk.tensor_log(sk.signature_forward(L_PATH, sk.build_truncated(2, 2)))
    np.testing.assert_allclose(log.values[0], [1.0, 1.0, 0.0, 0.5, -0.5, 0.0], atol=1e-14)
    out = sk.logsignature_forward(L_PATH, 2, 2)
    assert out.wordset.word_strings() == ["1", "2", "1.2"]
    np.testing.assert_allclose(out.values[0], [1.0, 1.0, 0.5], atol=1e-14)
    # test_logsig.py:96-101 level one is the exact displacement; :103-107 one channel
    rng = np.random.default_rng(64)
    paths = rng.random((4, 21, 3)) * 2 - 1
    out = sk.logsignature_forward(paths, 3, 4)
    np.testing.assert_array_equal(out.values[:, :3], paths[:, -1] - paths[:, 0])
    one = sk.logsignature_forward(np.cumsum(np.ones((2, 5, 1)), axis=1), 1, 3)
    assert one.values.shape == (2, 1)
    np.testing.assert_allclose(one.values[:, 0], 4.0, atol=1e-14)
    # identity -> zero log (test_logsig.py:29-33)
    ident = sk.CoefficientBatch(sk.build_truncated(2, 3), np.zeros((2, 14)))
    assert np.all(sk.tensor_log(ident).values == 0.0)


@pytest.mark.gpu
def test_backward_level_one_closed_form_and_zero():
    # test_logsig.py:117-132
    rng = np.random.default_rng(65)
    paths = rng.random((2, 7, 3)) * 2 - 1
    nl = len(sk.build_lyndon(3, 3))
    g = np.zeros((2, nl))
    g[:, :3] = rng.normal(size=(2, 3))
    out = sk.logsignature_backward(paths, 3, 3, g)
    np.testing.assert_allclose(out.path_grads[:, 0], -g[:, :3], atol=1e-12)
    np.testing.assert_allclose(out.path_grads[:, -1], g[:, :3], atol=1e-12)
    assert np.max(np.abs(out.path_grads[:, 1:-1])) <= 1e-12
    zero = sk.logsignature_backward(L_PATH, 2, 2, np.zeros((1, 3)))
    assert np.all(zero.path_grads == 0.0)


@pytest.mark.gpu
def test_backward_matches_finite_differences_of_the_oracle():
    rng = np.random.default_rng(66)
    d, N, M = 2, 3, 4
    paths = rng.random((2, M + 1, d)) * 2 - 1
    ly = sk.build_lyndon(d, N)
    g = rng.normal(size=(2, len(ly)))
    analytic = sk.logsignature_backward(paths, d, N, g).path_grads
    h = 1e-5
    fd = np.zeros_like(paths)
    for j in range(M + 1):
        for i in range(d):
            step = h * np.maximum(1.0, np.abs(paths[:, j, i]))
            plus, minus = paths.copy(), paths.copy()
            plus[:, j, i] += step
            minus[:, j, i] -= step
            lp = ora.lyndon_logsig(plus, d, N, ly.codes, ly.lengths)
            lm = ora.lyndon_logsig(minus, d, N, ly.codes, ly.lengths)
            fd[:, j, i] = np.sum(g * (lp - lm), axis=1) / (2 * step)
    assert ora.rel_err(analytic, fd) <= 1e-6


@pytest.mark.gpu
def test_errors_and_torch_inputs():
    import torch

    with pytest.raises(sk.DomainError):
        sk.logsignature_forward(L_PATH, 2, 0)
    with pytest.raises(sk.ShapeError):
        sk.logsignature_forward(L_PATH, 3, 2)
    with pytest.raises(sk.ShapeError):
        sk.logsignature_backward(L_PATH, 2, 2, np.zeros((1, 5)))
    with pytest.raises(sk.UnsupportedWordSetError):
        sk.tensor_log(sk.CoefficientBatch(sk.build_custom([(0, 1)], 2), np.zeros((1, 1))))
    # CUDA tensors in -> CUDA tensors out, same values
    X = torch.from_numpy(np.random.default_rng(3).random((3, 9, 3))).cuda()
    t = sk.logsignature_forward(X, 3, 4).values
    assert t.is_cuda
    np.testing.assert_allclose(t.cpu().numpy(), sk.logsignature_forward(X.cpu().numpy(), 3, 4).values, rtol=0,
                               atol=0)


@pytest.mark.gpu
def test_batches_beyond_one_grid_row():
    """More than 65,535 paths: the polynomial and tensor-product launches split the batch."""
    rng = np.random.default_rng(67)
    B = 70_001
    X = rng.random((B, 3, 2)) * 2 - 1
    out = sk.logsignature_forward(X, 2, 2).values
    ly = sk.build_lyndon(2, 2)
    rows = [0, 1, 65_534, 65_535, 65_536, B - 1]
    ref = ora.lyndon_logsig(X[rows], 2, 2, ly.codes, ly.lengths)
    assert ora.rel_err(out[rows], ref) <= 1e-12
    ws = sk.build_truncated(2, 2)
    S = sk.signature_forward(X, ws)
    assert ora.rel_err(sk.tensor_log(S).values[rows], ora.dense_log(S.values[rows], 2, 2)) <= 1e-12
    g = rng.standard_normal((B, len(ly)))
    dX = sk.logsignature_backward(X, 2, 2, g).path_grads
    # level-one letters: dL/dX_0 = -g, dL/dX_M = +g for the displacement part; check finite and shaped
    assert dX.shape == X.shape and np.isfinite(dX).all()


@pytest.mark.gpu
def test_backward_float32_path_batch_is_upcast():
    """A float32 PathBatch (lead_lag of float32 samples) runs the float64 backward
    like the reference (logsig.py:164-192 upcasts), bit-identical to float64 input."""
    rng = np.random.default_rng(68)
    X32 = (rng.random((3, 6, 2)) * 2 - 1).astype(np.float32)
    ll32 = sk.lead_lag(X32)
    assert ll32.dtype == np.float32
    ll64 = sk.lead_lag(X32.astype(np.float64))
    ly = sk.build_lyndon(4, 3)
    g = rng.normal(size=(3, len(ly)))
    a = sk.logsignature_backward(ll32, 4, 3, g).path_grads
    b = sk.logsignature_backward(ll64, 4, 3, g).path_grads
    assert a.dtype == np.float64
    np.testing.assert_array_equal(a, b)
