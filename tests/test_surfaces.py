"""Path transforms and scikit-learn surfaces over the GPU path.

Mirrors /root/reference/pkg/tests/test_transforms.py and test_estimators.py:
the same cases, with the dense oracle (oracle/oracle.py) as the checker.
"""

import numpy as np
import pytest

import paper_2602_24066_b200 as sk
from oracle import oracle as ora


def random_paths(rng, B, M, d):
    return rng.random((B, M + 1, d)) * 2.0 - 1.0


# -- CPU: transforms are data layout -------------------------------------------------------


def test_lead_lag_points_example():
    out = sk.lead_lag(np.array([[[0.0], [1.0], [3.0]]]))
    np.testing.assert_array_equal(out.samples, [[[0, 0], [0, 1], [1, 1], [1, 3], [3, 3]]])
    assert out.base_d == 1 and (out.B, out.M, out.d) == (1, 4, 2)


def test_lead_lag_constant_even_points_and_errors():
    assert np.all(sk.lead_lag(np.ones((2, 4, 3)) * 2.5).samples == 2.5)
    out = sk.lead_lag(random_paths(np.random.default_rng(70), 2, 5, 3))
    np.testing.assert_array_equal(out.samples[:, 0::2, :3], out.samples[:, 0::2, 3:])
    with pytest.raises(sk.DomainError):
        sk.lead_lag(np.zeros((1, 1, 2)))


def test_time_reverse():
    np.testing.assert_array_equal(sk.time_reverse(np.array([[[1.0], [2.0], [3.0]]])).samples, [[[3.0], [2.0], [1.0]]])
    p = random_paths(np.random.default_rng(73), 2, 5, 3)
    np.testing.assert_array_equal(sk.time_reverse(sk.time_reverse(p)).samples, p)


def test_estimator_params_without_device():
    from sklearn.base import clone

    est = sk.SignatureFeatures(word_set="anisotropic", gamma=[1, 2], r=3.0)
    assert clone(est).get_params()["gamma"] == [1, 2]
    assert clone(sk.WindowedSignatureFeatures(windows=[(0, 3)], depth=2)).get_params()["windows"] == [(0, 3)]
    with pytest.raises(sk.ShapeError):
        sk.SignatureFeatures().fit(np.zeros((4, 10)))


# -- GPU -----------------------------------------------------------------------------------


@pytest.mark.gpu
def test_lead_lag_signatures():
    rng = np.random.default_rng(71)
    out = sk.lead_lag(np.array([[[0.0], [1.0]]]))
    sig = sk.signature_forward(out, sk.build_custom([(0, 1), (1, 0)], 2))
    assert sig.values[0, 0] - sig.values[0, 1] == pytest.approx(-1.0, abs=1e-15)
    for d in (1, 2, 3):
        paths = random_paths(rng, 3, 8, d)
        ws = sk.build_truncated(2 * d, 2)
        sig = sk.signature_forward(sk.lead_lag(paths), ws)
        qv = np.sum(np.diff(paths, axis=1) ** 2, axis=1)
        for i in range(d):
            a = sig.values[:, ws.index_of(sk.encode_word((i, d + i), 2 * d))]
            b = sig.values[:, ws.index_of(sk.encode_word((d + i, i), 2 * d))]
            np.testing.assert_allclose(a - b, -qv[:, i], rtol=1e-12)
    paths = random_paths(np.random.default_rng(72), 2, 6, 2)
    ll = sk.lead_lag(paths)
    ws = sk.build_truncated(4, 2)
    sig = sk.signature_forward(ll, ws)
    assert ora.rel_err(sig.values, ora.dense_signature(ll.samples, 4, 2)) <= 1e-12


@pytest.mark.gpu
def test_signature_of_reverse_is_inverse():
    paths = random_paths(np.random.default_rng(74), 3, 6, 2)
    ws = sk.build_truncated(2, 3)
    fwd = sk.signature_forward(paths, ws)
    rev = sk.signature_forward(sk.time_reverse(paths), ws)
    assert ora.rel_err(rev.values, sk.signature_inverse(fwd).values) <= 1e-10


@pytest.mark.gpu
def test_signature_features():
    from sklearn.linear_model import Ridge
    from sklearn.pipeline import Pipeline

    rng = np.random.default_rng(90)
    X = random_paths(rng, 4, 10, 2)
    est = sk.SignatureFeatures(depth=3).fit(X)
    np.testing.assert_array_equal(est.transform(X), sk.signature_forward(X, sk.build_truncated(2, 3)).values)
    assert ora.rel_err(est.transform(X), ora.dense_signature(X, 2, 3)) <= 1e-12
    est = sk.SignatureFeatures(depth=2).fit(np.zeros((2, 3, 2)))
    assert list(est.get_feature_names_out()) == ["1", "2", "1.1", "1.2", "2.1", "2.2"]
    est = sk.SignatureFeatures(depth=1, include_empty=True).fit(np.zeros((2, 3, 2)))
    out = est.transform(np.zeros((2, 3, 2)))
    assert out.shape == (2, 3) and np.all(out[:, 0] == 1.0) and est.get_feature_names_out()[0] == "e"
    assert sk.SignatureFeatures(word_set="anisotropic", gamma=[1, 2], r=3).fit(np.zeros((1, 4, 2))).transform(
        np.zeros((1, 4, 2))).shape == (1, 6)
    est = sk.SignatureFeatures(word_set="custom", words=["2.1", "1"]).fit(np.zeros((1, 4, 2)))
    assert list(est.get_feature_names_out()) == ["1", "2.1"]
    X = random_paths(np.random.default_rng(91), 3, 6, 2)
    est = sk.SignatureFeatures(depth=2, lead_lag=True).fit(X)
    np.testing.assert_array_equal(est.transform(X),
                                  sk.signature_forward(sk.lead_lag(X), sk.build_truncated(4, 2)).values)
    X = random_paths(np.random.default_rng(92), 2, 5, 2)
    est = sk.SignatureFeatures(word_set="leadlag_sparse", depth=2, lead_lag=True).fit(X)
    assert est.wordset_ == sk.build_leadlag_sparse(2, 2)
    assert est.transform(X).shape == (2, 10)
    est = sk.SignatureFeatures(depth=2).fit(np.zeros((1, 3, 2)))
    with pytest.raises(sk.ShapeError):
        est.transform(np.zeros((1, 3, 3)))
    X = random_paths(np.random.default_rng(93), 20, 15, 2)
    y = X[:, -1, 0] - X[:, 0, 0]
    pipe = Pipeline([("sig", sk.SignatureFeatures(depth=2)), ("reg", Ridge(alpha=1e-6))]).fit(X, y)
    assert pipe.score(X, y) > 0.99


@pytest.mark.gpu
def test_logsignature_and_windowed_features():
    X = random_paths(np.random.default_rng(94), 3, 8, 2)
    est = sk.LogSignatureFeatures(depth=3).fit(X)
    np.testing.assert_array_equal(est.transform(X), sk.logsignature_forward(X, 2, 3).values)
    assert list(sk.LogSignatureFeatures(depth=3).fit(np.zeros((1, 3, 2))).get_feature_names_out()) == [
        "1", "2", "1.2", "1.1.2", "1.2.2"]
    X = random_paths(np.random.default_rng(95), 2, 10, 2)
    est = sk.WindowedSignatureFeatures(windows=[(0, 5), (5, 10)], depth=2).fit(X)
    out = est.transform(X)
    assert out.shape == (2, 12)
    ws = sk.build_truncated(2, 2)
    np.testing.assert_array_equal(out[:, :6], sk.signature_forward(X[:, :6], ws).values)
    np.testing.assert_array_equal(out[:, 6:], sk.signature_forward(X[:, 5:], ws).values)
    est = sk.WindowedSignatureFeatures(windows=[(0, 2)], depth=1).fit(np.zeros((1, 3, 2)))
    assert list(est.get_feature_names_out()) == ["0:2|1", "0:2|2"]


@pytest.mark.gpu
def test_features_on_cuda_tensors():
    """The transformers also take CUDA tensors and keep the features on the device."""
    import torch

    X = random_paths(np.random.default_rng(96), 3, 9, 2)
    Xt = torch.from_numpy(X).cuda()
    est = sk.SignatureFeatures(depth=3).fit(Xt)
    out = est.transform(Xt)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    np.testing.assert_array_equal(out.cpu().numpy(), sk.SignatureFeatures(depth=3).fit(X).transform(X))
    wt = sk.WindowedSignatureFeatures(windows=[(0, 4), (2, 9)], depth=2).fit(Xt).transform(Xt)
    wn = sk.WindowedSignatureFeatures(windows=[(0, 4), (2, 9)], depth=2).fit(X).transform(X)
    assert isinstance(wt, torch.Tensor)
    assert ora.rel_err(wt.cpu().numpy(), wn) <= 1e-12
    lt = sk.SignatureFeatures(depth=2, lead_lag=True).fit(Xt).transform(Xt)
    np.testing.assert_array_equal(lt.cpu().numpy(), sk.SignatureFeatures(depth=2, lead_lag=True).fit(X).transform(X))
