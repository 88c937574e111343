"""GPU parity of every kernel family on every kind of word set.

Kernel policies (sigb_set_kernel_policy): 0 = auto (truncated > generated
for small sparse sets > fragment > level; a generated kernel that is still
compiling in the background is served by the fragment kernels), 1 =
level-synchronous trie kernels, 2 = register-resident fragment kernels, 4 =
word-set specialised generated kernels (NVRTC, compiled synchronously).  Each family is checked against the C oracle (a restatement of the
reference numba kernels pinned to the reference's golden vectors) and the
golden vectors themselves, on the BASELINE configs' own word sets and on
random tries (prefix-closed and not), with the north_star tolerances:
fp64 <= 1e-10, fp32 <= 1e-4 relative to the fp64 oracle.
"""

import numpy as np
import pytest
import torch

import paper_2602_24066_b200 as sk
from paper_2602_24066_b200 import _lib
from oracle import oracle as ora
from tests.configs import CONFIGS, brownian, build_wordset

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


@pytest.fixture(params=[0, 1, 2, 4], ids=["auto", "level", "fragment", "generated"])
def policy(request):
    _lib.set_kernel_policy(request.param)
    yield request.param
    _lib.set_kernel_policy(0)


def random_trie(rng, d, depth, n, closed=True):
    words = [(int(rng.integers(d)),)]
    seen = set(words)
    tries = 0
    while len(words) < n and tries < 50 * n:
        tries += 1
        p = words[int(rng.integers(len(words)))]
        if len(p) >= depth:
            continue
        c = p + (int(rng.integers(d)),)
        if c not in seen:
            seen.add(c)
            words.append(c)
    if closed:
        for w in list(words):
            for k in range(1, len(w)):
                if w[:k] not in seen:
                    seen.add(w[:k])
                    words.append(w[:k])
    else:  # drop a few interior prefixes: the plan must compute but not emit them
        words = [w for i, w in enumerate(words) if len(w) == depth or i % 3]
    return sk.build_custom(words, d)


def check_set(ws, policy, B=3, L=12, seed=0):
    d = ws.d
    X = brownian(seed, B, L, d)
    plan = ws.plan()
    if policy == 2 and not plan.uses_fragments:
        pytest.skip("no fragment shape for this set")
    if policy == 4 and plan.kernel_kind != 4:
        pytest.skip("set too large for generated kernels")
    ref = ora.forward(X, ws.codes, ws.lengths, d)
    out = sk.signature_forward(X, ws).values
    assert ora.rel_err(out, ref) <= TOL64
    g = np.random.default_rng(seed + 1).standard_normal((B, len(ws)))
    _, dref = ora.backward(X, ws.codes, ws.lengths, d, g)
    res = sk.signature_backward(X, ws, g)
    assert ora.rel_err(res.path_grads, dref) <= TOL64
    X32 = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
    S32 = sk.signature(X32, ws)
    S32.backward(torch.from_numpy(g).float().cuda())
    assert ora.rel_err(S32.detach().cpu().numpy(), ref) <= TOL32
    assert ora.rel_err(X32.grad.cpu().numpy(), dref) <= TOL32


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_configs_every_family(golden_forward, golden_backward, policy, name):
    ws = build_wordset(name, sk)
    gf, gb = golden_forward, golden_backward
    tol = TOL64 if CONFIGS[name]["dtype"] == np.float64 else TOL32
    assert ora.rel_err(sk.signature_forward(gf[f"{name}/X"], ws).values, gf[f"{name}/S64"]) <= tol
    dX = sk.signature_backward(gb[f"{name}/X"], ws, gb[f"{name}/g"]).path_grads
    assert ora.rel_err(dX, gb[f"{name}/dX"]) <= TOL64
    X = torch.from_numpy(gb[f"{name}/X"].astype(np.float32)).cuda().requires_grad_(True)
    sk.signature(X, ws).backward(torch.from_numpy(gb[f"{name}/g"]).float().cuda())
    assert ora.rel_err(X.grad.cpu().numpy(), gb[f"{name}/dX"]) <= TOL32


def test_auto_routing():
    kinds = {n: build_wordset(n, sk).plan().kernel_kind for n in CONFIGS}
    assert kinds["c1"] == kinds["c2"] == kinds["c5"] == 1  # truncated kernels
    assert kinds["c3"] == 4  # generated kernels (sparse 2,048-word set)
    assert kinds["c4"] == 2  # fragment kernels


@pytest.mark.parametrize("seed", range(6))
def test_random_prefix_closed_tries(policy, seed):
    rng = np.random.default_rng(100 + seed)
    d = int(rng.integers(2, 18))
    depth = int(rng.integers(1, 7))
    ws = random_trie(rng, d, depth, int(rng.integers(5, 300)))
    check_set(ws, policy, B=int(rng.integers(1, 6)), L=int(rng.integers(2, 40)), seed=seed)


@pytest.mark.parametrize("seed", range(4))
def test_random_non_prefix_closed(policy, seed):
    rng = np.random.default_rng(200 + seed)
    ws = random_trie(rng, int(rng.integers(2, 9)), int(rng.integers(2, 6)), 60, closed=False)
    check_set(ws, policy, B=2, L=15, seed=seed)


@pytest.mark.parametrize("gamma,r", [((1.0, 2.0), 5.0), ((1.0, 1.0, 2.0, 3.0), 6.0), ((2.0, 1.0, 1.5), 4.5)])
def test_anisotropic_sets(policy, gamma, r):
    check_set(sk.build_anisotropic(sk.AnisotropyWeights(gamma, r)), policy, B=4, L=17)


@pytest.mark.parametrize("d,N", [(3, 6), (10, 3), (5, 4), (2, 7)])
def test_truncations_without_dedicated_kernel(policy, d, N):
    check_set(sk.build_truncated(d, N, include_empty=False), policy, B=2, L=10)


@pytest.mark.parametrize("B", [1, 2, 7, 33])
def test_fragment_batch_and_length_edges(B):
    _lib.set_kernel_policy(2)
    try:
        ws = build_wordset("c3", sk)
        for L in (1, 2, 17, 40):
            X = brownian(B + L, B, L, 16)
            out = sk.signature_forward(X, ws).values
            assert ora.rel_err(out, ora.forward(X, ws.codes, ws.lengths, 16)) <= TOL64
            g = np.random.default_rng(L).standard_normal((B, len(ws)))
            _, dref = ora.backward(X, ws.codes, ws.lengths, 16, g)
            assert ora.rel_err(sk.signature_backward(X, ws, g).path_grads, dref) <= TOL64
    finally:
        _lib.set_kernel_policy(0)


def test_fragment_include_empty_and_state():
    _lib.set_kernel_policy(2)
    try:
        ws = sk.build_custom([(0, 1, 1), (1,), (1, 0), (2, 2, 2, 2)], 3, include_empty=True)  # not prefix-closed
        X = brownian(9, 3, 11, 3)
        out = sk.signature_forward(X, ws).values
        assert np.all(out[:, 0] == 1.0)
        assert ora.rel_err(out[:, 1:], ora.forward(X, ws.codes, ws.lengths, 3)) <= TOL64
        g = np.random.default_rng(1).standard_normal((3, len(ws) + 1))
        _, dref = ora.backward(X, ws.codes, ws.lengths, 3, g[:, 1:])
        assert ora.rel_err(sk.signature_backward(X, ws, g).path_grads, dref) <= TOL64
        Xt = torch.from_numpy(X).cuda().requires_grad_(True)
        sk.signature(Xt, ws).backward(torch.from_numpy(g).cuda())
        assert ora.rel_err(Xt.grad.cpu().numpy(), dref) <= TOL64
    finally:
        _lib.set_kernel_policy(0)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_fragment_deterministic_bitwise(name):
    ws = build_wordset(name, sk)
    cfg = CONFIGS[name]
    X = torch.from_numpy(brownian(3, 16, 65, cfg["d"]).astype(np.float32)).cuda()
    g = torch.randn(16, len(ws), device="cuda")
    res = []
    for _ in range(2):
        Xr = X.clone().requires_grad_(True)
        S = sk.signature(Xr, ws)
        S.backward(g)
        res.append((S.detach().cpu().numpy(), Xr.grad.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_properties(name):
    """Full BASELINE batch and length: sum_j dX_j = 0 per path and channel (telescoping),
    and a fp64 oracle spot check of S and dX on the first and last path."""
    cfg = CONFIGS[name]
    ws = build_wordset(name, sk)
    B, L, d = cfg["B"], cfg["L"], cfg["d"]
    gen = torch.Generator(device="cuda").manual_seed(5)
    X = torch.cumsum(torch.randn(B, L, d, device="cuda", generator=gen) / np.sqrt(L - 1), dim=1)
    X[:, 0] = 0
    Xr = X.clone().requires_grad_(True)
    S = sk.signature(Xr, ws)
    g = torch.randn(B, len(ws), device="cuda", generator=gen)
    S.backward(g)
    dX = Xr.grad
    scale = dX.abs().amax(dim=1).clamp_min(1.0)
    assert float((dX.sum(dim=1) / scale).abs().max()) <= 1e-3
    for b in (0, B - 1):
        x = X[b:b + 1].double().cpu().numpy()
        ref = ora.forward(x, ws.codes, ws.lengths, d)
        assert ora.rel_err(S[b:b + 1].detach().cpu().numpy(), ref) <= TOL32
        _, dref = ora.backward(x, ws.codes, ws.lengths, d, g[b:b + 1].double().cpu().numpy())
        assert ora.rel_err(dX[b:b + 1].cpu().numpy(), dref) <= TOL32


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_windows_every_family(policy, name):
    """signature_windows (reference sigcore.py:242-263) on each kernel family: (path, window)
    pairs run as virtual paths; windows of different lengths share a CTA."""
    ws = build_wordset(name, sk)
    d = ws.d
    X = brownian(7, 3, 40, d)
    pairs = np.array([[0, 39], [5, 6], [10, 30], [0, 1], [38, 39], [3, 20], [1, 39]])
    outs = sk.signature_windows(X, ws, sk.WindowSpec(pairs))
    ref = ora.windows(X, ws.codes, ws.lengths, d, pairs)
    assert len(outs) == len(pairs)
    for k, o in enumerate(outs):
        assert ora.rel_err(o.values, ref[:, k]) <= TOL64, k
    # a whole-path window equals the forward signature bit for bit when both run the
    # same kernel family (level-slot / generated plans have no windowed form; windows
    # run on the fragment kernels)
    if ws.plan().kernel_kind not in (3, 4):
        assert np.array_equal(outs[0].values, sk.signature_forward(X, ws).values)
    else:
        assert ora.rel_err(outs[0].values, sk.signature_forward(X, ws).values) <= TOL64
    X32 = torch.from_numpy(X.astype(np.float32)).cuda()
    outs32 = sk.signature_windows(X32, ws, sk.WindowSpec(pairs))
    for k, o in enumerate(outs32):
        assert ora.rel_err(o.cpu().numpy() if isinstance(o, torch.Tensor) else o.values.cpu().numpy(),
                           ref[:, k]) <= TOL32, k


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_backward_memory_contract(name):
    """Memory-lean backward (reference test_acceptance.py:293-308): beyond its inputs, its
    outputs and the per-step gradient partials (B x parts x M x d, the size class of dX),
    the backward allocates nothing that grows with M -- no per-step signature trajectory."""
    ws = build_wordset(name, sk)
    d = ws.d
    plan = ws.plan()
    extra = []
    for L in (101, 4001):
        X = torch.from_numpy(brownian(1, 4, L, d).astype(np.float32)).cuda()
        S = torch.empty((4, len(ws)), device="cuda")
        plan.forward(X, S, 0, False)
        g = torch.randn(4, len(ws), device="cuda")
        dX = torch.empty_like(X)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        plan.backward(X, S, 0, False, g, 0, 0, dX)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base
        work = plan.workspace_bytes(torch.float32, 4, L, 0)
        assert work <= 64 * 4 * (L - 1) * d * 4  # partials: at most 64 parts x dX
        extra.append(peak - work)
    assert extra[1] <= extra[0] + (1 << 20), extra  # independent of M (1 MiB slack for the allocator)


@pytest.mark.gpu
@pytest.mark.parametrize("d,misaligned", [(16, False), (16, True), (10, False)])
def test_generated_kernels_many_path_blocks(d, misaligned):
    """Several 32-path blocks per task group (persistent claiming, lockstep slots
    with an idle slot at the tail), partial chunks, bulk-copy staging (d*4 % 16 == 0)
    and its element-copy fallback (d = 10, or a sample pointer off 16-byte alignment)."""
    _lib.set_kernel_policy(4)
    try:
        rng = np.random.default_rng(300 + d)
        ws = random_trie(rng, d, 4, 220)
        assert ws.plan().kernel_kind == 4
        B, L = 101, 45
        X = brownian(7, B, L, d)
        g = np.random.default_rng(8).standard_normal((B, len(ws)))
        ref = ora.forward(X, ws.codes, ws.lengths, d)
        _, dref = ora.backward(X, ws.codes, ws.lengths, d, g)
        flat = torch.empty(B * L * d + 1, dtype=torch.float32, device="cuda")
        X32 = (flat[1:] if misaligned else flat[:-1]).view(B, L, d)
        X32.copy_(torch.from_numpy(X.astype(np.float32)))
        X32.requires_grad_(True)
        S32 = sk.signature(X32, ws)
        S32.backward(torch.from_numpy(g).float().cuda())
        assert ora.rel_err(S32.detach().cpu().numpy(), ref) <= TOL32
        assert ora.rel_err(X32.grad.cpu().numpy(), dref) <= TOL32
        assert ora.rel_err(sk.signature_forward(X, ws).values, ref) <= TOL64
        assert ora.rel_err(sk.signature_backward(X, ws, g).path_grads, dref) <= TOL64
    finally:
        _lib.set_kernel_policy(0)


@pytest.mark.parametrize("d,N,B,L,force", [(4, 4, 4, 5001, False), (4, 6, 2, 4101, False), (8, 4, 5, 300, True),
                                            (16, 4, 3, 200, True), (4, 4, 32, 128, True)])
def test_parallel_in_time_forward(d, N, B, L, force, monkeypatch):
    """Small batches of long paths on full truncations run as T windows per path joined by a
    tree of truncated tensor products (signature.py _scan_forward; Chen's identity, reference
    sigcore.py:321-334): same values as the oracle (fp64 1e-10, fp32 1e-4) and as the
    sequential sweep (SIGB_SCAN=0), bitwise reproducible."""
    from paper_2602_24066_b200.signature import _scan_segments

    if force:
        monkeypatch.setenv("SIGB_SCAN", "2")
    ws = sk.build_truncated(d, N)
    X = brownian(60 + d, B, L, d)
    assert _scan_segments(ws.plan(), ws, B, L - 1) > 1
    ref = ora.forward(X, ws.codes, ws.lengths, d)
    out = sk.signature_forward(X, ws).values
    assert ora.rel_err(out, ref) <= TOL64
    assert np.array_equal(out, sk.signature_forward(X, ws).values)
    X32 = X.astype(np.float32)
    out32 = sk.signature_forward(X32, ws).values
    ref32 = ora.forward(X32.astype(np.float64), ws.codes, ws.lengths, d)
    assert ora.rel_err(out32, ref32) <= TOL32
    monkeypatch.setenv("SIGB_SCAN", "0")
    assert ora.rel_err(sk.signature_forward(X, ws).values, out) <= TOL64
    ws_e = sk.build_truncated(d, N, include_empty=True)
    monkeypatch.setenv("SIGB_SCAN", "2" if force else "1")
    oe = sk.signature_forward(X, ws_e).values
    assert np.all(oe[:, 0] == 1.0) and ora.rel_err(oe[:, 1:], ref) <= TOL64
