"""Host-side logic on CPU: word encodings, builders, descriptor, validation.

Known answers are the reference's own examples (reference tests/test_words.py,
tests/test_wordsets.py) and the fingerprints/hashes of the five BASELINE word
sets recorded from the reference builders in tests/golden/meta.json.  No
device work happens here.
"""

import hashlib
import itertools

import numpy as np
import pytest

import paper_2602_24066_b200 as sk
from paper_2602_24066_b200.wordcodes import EMPTY_WORD
from tests.configs import CONFIGS, build_wordset


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def letter_set(ws):
    return {sk.decode_word(w, ws.d) for w in ws.words}


# -- words.py (reference words.py:84-206) -------------------------------------------------


def test_encode_decode_examples():
    W = sk.Word
    assert sk.encode_word((1, 0), 2) == W(2, 2)
    assert sk.encode_word((), 5) == W(0, 0)
    assert sk.encode_word((1, 1), 3) == W(2, 4)
    assert sk.decode_word(W(3, 5), 2) == (1, 0, 1)
    assert sk.decode_word(W(0, 0), 7) == ()
    with pytest.raises(sk.InvalidLetterError):
        sk.encode_word((0, 2), 2)
    with pytest.raises(sk.CorruptWordError):
        sk.decode_word(W(2, 4), 2)


def test_capacity():
    assert sk.max_word_length(2) == 64
    assert sk.max_word_length(4) == 32
    assert sk.max_word_length(1) == 64
    with pytest.raises(sk.CapacityError):
        sk.encode_word((1,) * 65, 2)
    with pytest.raises(sk.CapacityError):
        sk.concat_code(sk.Word(40, 0), sk.Word(40, 0), 3)


def test_prefix_suffix_concat():
    W = sk.Word
    w = W(3, 5)
    assert sk.concat_code(W(1, 1), W(2, 1), 2) == w
    assert sk.concat_code(EMPTY_WORD, W(2, 3), 2) == W(2, 3)
    assert sk.concat_code(W(1, 2), W(1, 0), 3) == W(2, 6)
    assert sk.prefix_code(w, 1, 2) == W(1, 1)
    assert sk.prefix_code(w, 0, 2) == EMPTY_WORD
    assert sk.suffix_code(w, 2, 2) == W(2, 1)
    assert sk.suffix_code(W(2, 6), 1, 3) == W(1, 0)
    with pytest.raises(sk.WordRangeError):
        sk.prefix_code(W(2, 1), 3, 2)
    rng = np.random.default_rng(9)
    for _ in range(100):
        d = int(rng.integers(2, 8))
        n = int(rng.integers(0, 10))
        w = sk.encode_word(tuple(int(x) for x in rng.integers(0, d, n)), d)
        for k in range(n + 1):
            assert sk.concat_code(sk.prefix_code(w, k, d), sk.suffix_code(w, n - k, d), d) == w


def test_code_order_is_lexicographic():
    rng = np.random.default_rng(8)
    for _ in range(100):
        d = int(rng.integers(2, 7))
        n = int(rng.integers(1, 9))
        a = tuple(int(x) for x in rng.integers(0, d, n))
        b = tuple(int(x) for x in rng.integers(0, d, n))
        assert (a < b) == (sk.encode_word(a, d).code < sk.encode_word(b, d).code)


def test_packing():
    assert sk.pack_letters(sk.encode_word((1, 0, 1), 2), 2, 2).bits == 17
    assert sk.pack_letters(EMPTY_WORD, 3, 5).bits == 0
    assert sk.pack_letters(sk.encode_word((3,), 4), 2, 4).bits == 3
    with pytest.raises(sk.CapacityError):
        sk.pack_letters(sk.encode_word((1,), 4), 1, 4)
    rng = np.random.default_rng(10)
    for _ in range(100):
        d = int(rng.integers(1, 11))
        b = sk.Alphabet(d).bits_per_letter
        n = int(rng.integers(0, 64 // b + 1))
        if n > sk.max_word_length(d):
            continue
        w = sk.encode_word(tuple(int(x) for x in rng.integers(0, d, n)), d)
        assert sk.unpack_letters(sk.pack_letters(w, b, d)) == sk.decode_word(w, d)


def test_word_strings():
    assert sk.word_to_string(sk.encode_word((0, 1, 1), 2), 2) == "1.2.2"
    assert sk.word_from_string("1.2.2", 2) == sk.encode_word((0, 1, 1), 2)
    assert sk.word_to_string(EMPTY_WORD, 4) == "e"
    for bad in ("1.3", "0.1", "1..2"):
        with pytest.raises(sk.InvalidLetterError):
            sk.word_from_string(bad, 2)


# -- wordsets.py builders (reference wordsets.py:278-511) ----------------------------------


def test_truncated_dimensions():
    assert len(sk.build_truncated(6, 3)) == 258
    assert len(sk.build_truncated(8, 6)) == 299_592
    assert letter_set(sk.build_truncated(2, 1)) == {(0,), (1,)}
    with pytest.raises(sk.DomainError):
        sk.build_truncated(2, 0)
    with pytest.raises(sk.CapacityError):
        sk.build_truncated(2, 65)


def test_anisotropic_examples():
    ws = sk.build_anisotropic(sk.AnisotropyWeights((1.0, 2.0), 3.0))
    assert letter_set(ws) == {(0,), (1,), (0, 0), (0, 1), (1, 0), (0, 0, 0)}
    for d, N in [(2, 3), (3, 2)]:
        assert sk.build_anisotropic(sk.AnisotropyWeights((1.0,) * d, float(N))) == sk.build_truncated(d, N)
    assert letter_set(sk.build_anisotropic(sk.AnisotropyWeights((1.0, 5.0), 1.0))) == {(0,)}
    gamma, r = (1.0, 2.0, 3.0), 5.0
    ws = sk.build_anisotropic(sk.AnisotropyWeights(gamma, r))
    brute = {w for n in range(1, 6) for w in itertools.product(range(3), repeat=n) if sum(gamma[i] for i in w) <= r}
    assert letter_set(ws) == brute
    with pytest.raises(sk.DomainError):
        sk.AnisotropyWeights((1.0, 0.0), 2.0)


def test_custom_canonical_and_dedup():
    ws = sk.build_custom([(1, 0), (0,), (1, 0), (1,)], 2)
    assert [sk.decode_word(w, 2) for w in ws.words] == [(0,), (1,), (1, 0)]
    with pytest.raises(sk.DomainError):
        sk.build_custom([()], 2)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_wordsets_match_reference_fingerprints(golden_meta, name):
    m = golden_meta["wordsets"][name]
    ws = build_wordset(name, sk)
    assert len(ws) == m["W"]
    assert ws.max_len == m["max_len"]
    assert int(np.asarray(ws.lengths).sum()) == m["sum_len"]
    assert sha(ws.codes) == m["codes_sha"]
    assert sha(ws.lengths) == m["lengths_sha"]
    fp = hashlib.sha256(",".join(ws.word_strings()).encode()).hexdigest()[:16]
    assert fp == m["fingerprint"]


def test_descriptor():
    assert sk.wordset_from_descriptor({"type": "truncated", "d": 2, "depth": 2}) == sk.build_truncated(2, 2)
    ws = sk.wordset_from_descriptor({"type": "custom", "d": 2, "words": ["1.2", "2"]})
    assert letter_set(ws) == {(0, 1), (1,)}
    ws = sk.wordset_from_descriptor({"type": "graph", "d": 2, "depth": 2, "edges": [[1, 2]]})
    assert letter_set(ws) == {(0,), (1,), (0, 1)}
    assert len(sk.wordset_from_descriptor({"type": "anisotropic", "d": 2, "gamma": [1, 2], "r": 3})) == 6
    assert sk.wordset_from_descriptor({"type": "lyndon", "depth": 2}, default_d=3).d == 3
    with pytest.raises(sk.DomainError):
        sk.wordset_from_descriptor({"type": "nope", "d": 2})


# -- API validation happens before any device call (reference sigcore.py:36-88) ------------


def test_path_batch_validation():
    with pytest.raises(sk.ShapeError):
        sk.PathBatch(np.zeros((2, 3)))
    with pytest.raises(sk.DomainError):
        sk.PathBatch(np.full((1, 2, 2), np.nan))
    pb = sk.PathBatch(np.zeros((1, 2, 2), dtype=np.int32))
    assert pb.samples.dtype == np.float64
    assert sk.PathBatch(np.full((1, 2, 2), np.nan), allow_nonfinite=True).M == 1


def test_window_spec_validation():
    with pytest.raises(sk.WindowError):
        sk.WindowSpec(np.array([[2, 1]]))
    with pytest.raises(sk.WindowError):
        sk.WindowSpec(np.zeros((0, 2)))
    with pytest.raises(sk.WindowError):
        sk.WindowSpec(np.array([[0, 5]])).validate_for(3)


def test_no_cpu_fallback():
    """Without a CUDA device the compute entry points raise instead of computing on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    ws = sk.build_truncated(2, 2)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sk.signature_forward(np.zeros((1, 3, 2)), ws)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sk.signature_backward(np.zeros((1, 3, 2)), ws, np.ones((1, 6)))
