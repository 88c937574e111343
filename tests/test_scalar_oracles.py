"""The scalar math oracles of SURVEY.md 8(a) row a11, CPU only.

``segment_exp_coeff`` / ``horner_update`` (reference sigcore.py:169-195) and
``exp_coeff_grad`` / ``left_step`` / ``right_step`` / ``ReconstructionState``
(reference backward.py:46-127) are the closed forms the kernels must agree
with.  These tests follow the reference's own (pkg/tests/test_backward.py:26-124:
finite differences, identity, one-segment inversion, reconstruction at every
step to 1e-9), with the C oracle (oracle/, pinned to the reference's golden
vectors) standing in for the reference's numba ``signature_forward`` so they
run without a GPU.
"""

import math

import numpy as np
import pytest

import paper_2602_24066_b200 as sk
from oracle import oracle as ora
from paper_2602_24066_b200.wordcodes import EMPTY_WORD


def _fwd(paths, ws):
    return ora.forward(np.asarray(paths, dtype=np.float64), ws.codes, ws.lengths, ws.d)


def _random_paths(rng, B, M, d):
    X = np.zeros((B, M + 1, d))
    X[:, 1:] = np.cumsum(rng.normal(size=(B, M, d)) / np.sqrt(M), axis=1)
    return X


# -- exp_coeff_grad (backward.py:46-58) ----------------------------------------------------


def test_exp_coeff_grad_repeated_letter():
    # d/dx of x^2/2 is x
    assert sk.exp_coeff_grad((0.7, -0.3), sk.encode_word((0, 0), 2), 0) == pytest.approx(0.7)


def test_exp_coeff_grad_empty_word():
    assert sk.exp_coeff_grad((1.0, 2.0), EMPTY_WORD, 0) == 0.0


def test_exp_coeff_grad_mixed_letters():
    # d/dx of x*y/2 w.r.t. x is y/2
    assert sk.exp_coeff_grad((0.4, 0.9), sk.encode_word((0, 1), 2), 0) == pytest.approx(0.45)


def test_exp_coeff_grad_matches_finite_difference():
    rng = np.random.default_rng(0)
    for _ in range(40):
        d = int(rng.integers(1, 4))
        n = int(rng.integers(0, 5))
        w = sk.encode_word(tuple(int(x) for x in rng.integers(0, d, n)), d)
        delta = rng.normal(size=d)
        i = int(rng.integers(0, d))
        h = 1e-6
        dp, dm = delta.copy(), delta.copy()
        dp[i] += h
        dm[i] -= h
        fd = (sk.segment_exp_coeff(dp, w) - sk.segment_exp_coeff(dm, w)) / (2 * h)
        assert sk.exp_coeff_grad(delta, w, i) == pytest.approx(fd, abs=1e-8)


# -- segment_exp_coeff / horner_update (sigcore.py:169-195) -------------------------------


def test_segment_exp_coeff_is_one_segment_signature():
    """<exp(delta), w> is the signature of a one-segment path (reference test_sigcore.py:80-87)."""
    rng = np.random.default_rng(3)
    for d, N in ((2, 3), (3, 4), (4, 2)):
        ws = sk.build_truncated(d, N)
        delta = rng.normal(size=d)
        X = np.stack([np.zeros(d), delta])[None]
        S = _fwd(X, ws)[0]
        for j, w in enumerate(ws.words):
            assert sk.segment_exp_coeff(delta, w) == pytest.approx(S[j], rel=1e-13, abs=1e-15)
        assert sk.segment_exp_coeff(delta, EMPTY_WORD) == 1.0


def test_horner_update_is_one_chen_step():
    """horner_update(prefix values of w at t_j, delta_j, w) = S_{0,t_{j+1}}(w) (Alg. 1)."""
    rng = np.random.default_rng(4)
    d = 3
    X = _random_paths(rng, 1, 7, d)
    for letters in ((0,), (1, 2), (2, 0, 1), (1, 1, 0, 2)):
        pre = [letters[:k] for k in range(1, len(letters) + 1)]
        ws = sk.build_custom(pre, d)
        w = sk.encode_word(letters, d)
        for j in range(1, 7):
            before = _fwd(X[:, : j + 1], ws)[0]
            after = _fwd(X[:, : j + 2], ws)[0]
            prev = [1.0] + [before[ws.index_of(sk.encode_word(p, d))] for p in pre]
            got = sk.horner_update(prev, X[0, j + 1] - X[0, j], w)
            assert got == pytest.approx(after[ws.index_of(w)], rel=1e-12, abs=1e-14)
    with pytest.raises(sk.ShapeError):
        sk.horner_update([1.0, 0.0], np.zeros(2), sk.encode_word((0, 1), 2))


# -- left_step / right_step / ReconstructionState (backward.py:61-127) ----------------------


def test_right_step_one_from_identity():
    out = sk.right_step(np.array([1.0, 0.0, 0.0]), (0, 1), np.array([0.3, -0.8]))
    assert out[0] == 1.0
    assert out[1] == pytest.approx(-0.8)  # last letter is channel 1
    assert out[2] == pytest.approx(0.3 * -0.8 / 2)


def test_zero_increment_is_noop():
    letters = (0, 1, 0)
    state = np.array([1.0, 0.5, 0.25, 0.125])
    zero = np.zeros(2)
    np.testing.assert_array_equal(sk.left_step(state, letters, zero), state)
    np.testing.assert_array_equal(sk.right_step(state, letters, zero), state)


def test_left_step_inverts_one_segment():
    delta = np.array([0.6, -0.4])
    terminal = np.array([1.0, -0.4, 0.6 * -0.4 / 2])
    np.testing.assert_allclose(sk.left_step(terminal, (1, 0), delta), [1.0, 0.0, 0.0], atol=1e-15)


def test_full_right_recursion_reproduces_forward():
    rng = np.random.default_rng(1)
    d = 2
    paths = _random_paths(rng, 1, 6, d)
    letters = (0, 1, 1)
    ws = sk.build_custom([letters], d)
    state = np.zeros(4)
    state[0] = 1.0
    for j in range(5, -1, -1):
        state = sk.right_step(state, letters, paths[0, j + 1] - paths[0, j])
    assert state[3] == pytest.approx(_fwd(paths, ws)[0, 0], rel=1e-12)


def test_reconstruction_matches_forward_at_every_step():
    """The memory-lean backward's invariant: pulling S_{0,T} back by exp(-delta_j) gives the
    forward signature of samples 0..j, and the right state the signature of samples j..M,
    at every step to 1e-9 (reference test_backward.py:96-124)."""
    rng = np.random.default_rng(2)
    d, M = 3, 20
    paths = _random_paths(rng, 1, M, d)
    letters = (2, 0, 1)
    n = len(letters)
    prefixes = [letters[:k] for k in range(n + 1)]
    suffixes = [letters[n - k:] for k in range(n + 1)]
    ws_pref = sk.build_custom([p for p in prefixes if p], d)
    ws_suff = sk.build_custom([s for s in suffixes if s], d)
    pcol = [None] + [ws_pref.index_of(sk.encode_word(prefixes[k], d)) for k in range(1, n + 1)]
    scol = [None] + [ws_suff.index_of(sk.encode_word(suffixes[k], d)) for k in range(1, n + 1)]
    terminal = np.zeros(n + 1)
    terminal[0] = 1.0
    fwd = _fwd(paths, ws_pref)[0]
    for k in range(1, n + 1):
        terminal[k] = fwd[pcol[k]]
    state = sk.ReconstructionState.terminal(letters, terminal)
    for j in range(M - 1, -1, -1):
        state.step_back(paths[0, j + 1] - paths[0, j])
        left_fwd = _fwd(paths[:, : j + 1], ws_pref)[0]
        right_fwd = _fwd(paths[:, j:], ws_suff)[0]
        for k in range(1, n + 1):
            assert abs(state.left[k] - left_fwd[pcol[k]]) <= 1e-9
            assert abs(state.right[k] - right_fwd[scol[k]]) <= 1e-9
    np.testing.assert_allclose(state.left, [1, 0, 0, 0], atol=1e-9)


def test_gradient_identity_from_scalar_oracles():
    """Prop. 4.1 assembled from the scalar oracles equals the oracle
    backward: dL/d delta_j[i] = sum_w g_w sum_{k<=m} left_k(w) d<exp(delta_j), w[k:m]>/d delta[i] right(w[m:])."""
    rng = np.random.default_rng(9)
    d, M = 2, 5
    paths = _random_paths(rng, 1, M, d)
    words = [(0,), (1, 0), (0, 1, 1)]
    ws = sk.build_custom(words, d)
    g = rng.normal(size=(1, len(ws)))
    dinc, _ = ora.backward(paths, ws.codes, ws.lengths, d, g)
    want = np.zeros((M, d))
    for wi, w in enumerate(ws.words):
        letters = sk.decode_word(w, d)
        n = len(letters)
        pre = [letters[:k] for k in range(1, n + 1)]
        wsp = sk.build_custom(pre, d)
        term = np.zeros(n + 1)
        term[0] = 1.0
        S = _fwd(paths, wsp)[0]
        for k in range(1, n + 1):
            term[k] = S[wsp.index_of(sk.encode_word(letters[:k], d))]
        st = sk.ReconstructionState.terminal(letters, term)
        for j in range(M - 1, -1, -1):
            delta = paths[0, j + 1] - paths[0, j]
            right_after = st.right.copy()
            st.step_back(delta)
            for i in range(d):
                acc = 0.0
                for a in range(n + 1):          # split w = w[:a] . w[a:b] . w[b:]
                    for b in range(a, n + 1):
                        mid = sk.encode_word(letters[a:b], d)
                        acc += st.left[a] * sk.exp_coeff_grad(delta, mid, i) * right_after[n - b]
                want[j, i] += g[0, ws.index_of(w)] * acc
    np.testing.assert_allclose(dinc[0], want, rtol=1e-10, atol=1e-12)
    assert math.isfinite(float(np.abs(want).sum()))
