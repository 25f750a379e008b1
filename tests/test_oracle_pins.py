"""Pins for the oracle (CPU, no GPU): each test checks oracle/ against something other than itself —
published known-answer vectors, the paper's / SPEC's worked values, closed forms, library routines
(torch autograd on the dense special case), finite differences, identities and brute force."""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import OracleConfig, MARGIN_NONE, MARGIN_ARCFACE, MARGIN_COSFACE
from synth import w_rows_np, make_labels, make_features

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_values():
    vals = {}
    for line in open(os.path.join(GOLDEN, "paper_values.txt")):
        if line.startswith("#") or not line.strip():
            continue
        parts = line.split()
        vals[parts[0]] = parts[1:]
    return vals


# ---------------------------------------------------------------- Philox (R2)
def test_philox_known_answers():
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        out = oracle.philox4x32_10(*w[:6])
        assert [int(o) for o in out] == w[6:], line


def test_philox_matches_curand_header_definition_on_vector_input():
    # the vectorised form agrees element-wise with per-element scalar calls (vectorisation is not a
    # source of error), and distinct counters give distinct outputs
    ids = np.arange(1000, dtype=np.uint64)
    vec = oracle.class_key(ids, seed=5, step=3)
    sc = np.array([int(oracle.class_key(np.array([i], dtype=np.uint64), 5, 3)[0]) for i in range(0, 1000, 97)])
    assert np.array_equal(vec[::97].astype(np.int64), sc)
    assert len(np.unique(vec)) > 990


# ---------------------------------------------------------------- partition and budget
def test_shard_range_partitions_in_order():
    for C, k in [(10, 3), (85742, 8), (1000, 1), (7, 7), (360232, 4)]:
        pos = 0
        sizes = []
        for i in range(k):
            a, n = oracle.shard_range(C, k, i)
            assert a == pos
            pos += n
            sizes.append(n)
        assert pos == C and max(sizes) - min(sizes) <= 1
        assert sizes == sorted(sizes, reverse=True)


def test_budget_closed_forms_for_baseline_configs():
    g = _golden_values()
    for name, (spec, expect) in g.items():
        if not name.startswith("k_"):
            continue
        f = spec.split(",")
        C, k, r = int(f[0]), int(f[1]), float(f[2])
        rank = int(f[3]) if len(f) > 3 else 0
        _, Cl = oracle.shard_range(C, k, rank)
        assert oracle.sample_budget(r, Cl) == int(expect), name


def test_positives_example_spec():
    # labels [3,3,7], shard [0,10) -> {3,7}; disjoint shard -> {}
    assert oracle.positives([3, 3, 7], 0, 10).tolist() == [3, 7]
    assert oracle.positives([3, 7], 10, 10).tolist() == []


@pytest.mark.parametrize("C,k,B,r,mode", [
    (1000, 1, 64, 0.1, "uniform"), (997, 4, 16, 0.05, "uniform"), (200, 2, 64, 0.01, "stress"),
    (50, 2, 8, 1.0, "uniform"), (85742, 8, 128, 0.1, "uniform"),
])
def test_sampler_invariants(C, k, B, r, mode):
    ys = make_labels(3, 0, k, B, C, mode=mode, stress_range=max(2, C // k // 2))
    Y = np.concatenate(ys)
    for i in range(k):
        a, Cl = oracle.shard_range(C, k, i)
        idx, npos = oracle.sample_shard(Y, a, Cl, r, seed=11, step=2)
        P = oracle.positives(Y, a, Cl)
        assert npos == len(P)
        assert len(idx) == max(oracle.sample_budget(r, Cl), len(P))         # |S_i| = k_i exactly
        assert np.all(np.diff(idx) > 0)                                     # ascending, unique
        assert idx.min() >= a and idx.max() < a + Cl                       # inside the shard
        assert set(P.tolist()) <= set(idx.tolist())                         # PPRN: positives kept
        if r == 1.0:
            assert np.array_equal(idx, np.arange(a, a + Cl))                # r = 1: identity layout


def test_sampler_stress_all_labels_in_one_shard():
    C, k, B = 2000, 2, 64
    ys = make_labels(1, 0, k, B, C, mode="distinct")
    Y = np.concatenate([np.arange(0, 128)])  # 128 distinct labels all in shard 0, r*C_local = 10
    idx, npos = oracle.sample_shard(Y, 0, 1000, 0.01, seed=1, step=0)
    assert npos == 128 and len(idx) == 128 and np.array_equal(idx, np.arange(128))
    idx1, npos1 = oracle.sample_shard(Y, 1000, 1000, 0.01, seed=1, step=0)
    assert npos1 == 0 and len(idx1) == 10


def _bruteforce_select(U, h, n):
    # j is selected iff fewer than n elements u of U precede it in the (h_u, u) order: O(|U|^2) count.
    sel = []
    for jj, (hj, j) in enumerate(zip(h, U)):
        before = sum(1 for hu, u in zip(h, U) if (hu < hj) or (hu == hj and u < j))
        if before < n:
            sel.append(int(j))
    return sorted(sel)


def test_sampler_bruteforce_tiny_with_forced_ties(monkeypatch):
    rng = np.random.default_rng(0)
    for trial in range(30):
        C_local = int(rng.integers(5, 40))
        a = int(rng.integers(0, 1000))
        Y = rng.integers(a, a + C_local, size=int(rng.integers(0, 6)))
        r = float(rng.choice([0.1, 0.3, 0.5, 0.9]))
        # force many equal keys: keys drawn from a tiny alphabet
        forced = {}

        def fake_key(ids, seed, step):
            ids = np.asarray(ids, dtype=np.int64)
            return np.array([forced.setdefault(int(j), int(rng.integers(0, 3))) for j in ids], dtype=np.uint64)

        monkeypatch.setattr(oracle.pfc, "class_key", fake_key)
        idx, npos = oracle.sample_shard(Y, a, C_local, r, seed=0, step=0)
        P = np.unique(Y)
        U = np.array([j for j in range(a, a + C_local) if j not in set(P.tolist())], dtype=np.int64)
        n = max(math.ceil(r * C_local), len(P)) - len(P)
        h = [forced[int(j)] for j in U]
        expect = sorted(set(P.tolist()) | set(_bruteforce_select(U, h, n)))
        assert idx.tolist() == expect


def test_sampler_uniform_frequency():
    # SPEC.md:286-style Monte-Carlo: shard of 100, 10 positives, 9 negatives from 90 -> 10% each
    a, Cl = 0, 100
    Y = np.arange(10)
    r = 0.19                                            # ceil(19.0) = 19 = 10 positives + 9 negatives
    T = 20000
    counts = np.zeros(Cl)
    for step in range(T):
        idx, _ = oracle.sample_shard(Y, a, Cl, r, seed=1234, step=step)
        counts[idx] += 1
    freq = counts[10:] / T
    assert np.all(np.abs(freq - 0.1) < 0.012), (freq.min(), freq.max())
    assert np.all(counts[:10] == T)


def test_sampler_reproducible_and_partition_independent_keys():
    Y = np.array([5, 17, 17, 40])
    i1, _ = oracle.sample_shard(Y, 0, 64, 0.25, seed=9, step=4)
    i2, _ = oracle.sample_shard(Y, 0, 64, 0.25, seed=9, step=4)
    i3, _ = oracle.sample_shard(Y, 0, 64, 0.25, seed=9, step=5)
    assert np.array_equal(i1, i2) and not np.array_equal(i1, i3)
    # h_j depends on the global id only
    assert np.array_equal(oracle.class_key(np.arange(32, 64), 9, 4), oracle.class_key(np.arange(64), 9, 4)[32:])


# ---------------------------------------------------------------- normalisation and margins
def test_normalize_examples():
    v, n = oracle.normalize_rows([[3.0, 4.0]])
    assert np.allclose(v, [[0.6, 0.8]], atol=1e-15) and n[0] == 5.0
    v2, _ = oracle.normalize_rows([[1.0, 0.0], [0.0, 2.0]])
    assert np.array_equal(v2, [[1.0, 0.0], [0.0, 1.0]])
    rng = np.random.default_rng(1)
    a = rng.standard_normal((20, 7)) * 7.3
    b, _ = oracle.normalize_rows(a)
    c, _ = oracle.normalize_rows(b)
    assert np.allclose(b, c, atol=1e-12)                                   # idempotent


def test_margin_values():
    g = _golden_values()
    s = 64.0
    assert s * oracle.margin_phi(0.9, MARGIN_COSFACE, 0.4) == pytest.approx(float(g["cosface_s64_m04_c09"][0]), abs=1e-12)
    assert s * oracle.margin_phi(math.cos(0.3), MARGIN_ARCFACE, 0.5) == pytest.approx(float(g["arcface_s64_m05_theta03"][0]), abs=1e-12)
    th = float(g["arcface_threshold_m05"][0])
    off = float(g["arcface_fallback_offset_m05"][0])
    assert math.cos(math.pi - 0.5) == pytest.approx(th, abs=1e-15)
    c = th - 0.01
    assert oracle.margin_phi(c, MARGIN_ARCFACE, 0.5) == pytest.approx(c - off, abs=1e-15)
    assert oracle.margin_phi(0.3, MARGIN_NONE, 0.5) == 0.3
    # zero margin is the identity (SPEC.md cosface m=0)
    cs = np.linspace(-1, 1, 11)
    assert np.allclose(oracle.margin_phi(cs, MARGIN_COSFACE, 0.0), cs)
    assert np.allclose(oracle.margin_phi(cs, MARGIN_ARCFACE, 0.0), cs, atol=1e-15)
    # monotonicity: margin makes the target strictly smaller on theta in (0, pi - m)
    th_grid = np.linspace(0.01, math.pi - 0.51, 50)
    assert np.all(oracle.margin_phi(np.cos(th_grid), MARGIN_ARCFACE, 0.5) < np.cos(th_grid))


def test_margin_derivative_matches_central_differences():
    for mt, m in [(MARGIN_ARCFACE, 0.5), (MARGIN_COSFACE, 0.4), (MARGIN_ARCFACE, 0.2)]:
        cs = np.linspace(-0.85, 0.98, 41)
        h = 1e-6
        fd = (oracle.margin_phi(cs + h, mt, m) - oracle.margin_phi(cs - h, mt, m)) / (2 * h)
        assert np.allclose(oracle.margin_dphi(cs, mt, m), fd, rtol=1e-6, atol=1e-7)


# ---------------------------------------------------------------- loss / softmax closed forms
def _orthogonal_case(C, margin_type=MARGIN_NONE, m=0.0, s=1.0, k=1):
    # d = C + 1: x = e_0, W rows e_1..e_C -> all cosines 0
    d = C + 1
    W = np.zeros((C, d)); W[np.arange(C), np.arange(1, C + 1)] = 1.0
    cfg = OracleConfig(num_classes=C, dim=d, batch=1, world_size=k, sample_rate=1.0, scale=s,
                       margin_type=margin_type, margin=m)
    xs = [np.eye(1, d) for _ in range(k)]
    ys = [np.array([0]) for _ in range(k)]
    return cfg, xs, ys, (lambda ids: W[np.asarray(ids)])


def test_uniform_loss_is_log_C():
    cfg, xs, ys, wr = _orthogonal_case(6)
    out = oracle.forward_backward(cfg, xs, ys, wr, keep_intermediates=True)
    assert out["loss"] == pytest.approx(math.log(6), abs=1e-14)
    assert np.allclose(out["prob"], 1 / 6)
    # CosFace on the same geometry: closed form log(e^{-s m} + (C-1)) + s m
    cfg, xs, ys, wr = _orthogonal_case(6, MARGIN_COSFACE, 0.4, 64.0)
    out = oracle.forward_backward(cfg, xs, ys, wr)
    assert out["loss"] == pytest.approx(math.log(math.exp(-25.6) + 5) + 25.6, abs=1e-12)


def test_two_equal_logits_over_two_ranks_and_grad_example():
    # SPEC.md:199 (two equal logits split across 2 workers -> 0.5) and SPEC.md:208 ([.5,.5] -> [-.5,.5])
    cfg, xs, ys, wr = _orthogonal_case(2, k=1)
    out = oracle.forward_backward(cfg, xs, ys, wr, keep_intermediates=True)
    assert np.allclose(out["prob"], [[0.5, 0.5]])
    assert np.allclose(out["Gc"], [[-0.5, 0.5]])
    cfg2 = OracleConfig(num_classes=2, dim=3, batch=1, world_size=2, sample_rate=1.0, scale=1.0,
                        margin_type=MARGIN_NONE)
    W = np.array([[0, 1.0, 0], [0, 0, 1.0]])
    out2 = oracle.forward_backward(cfg2, [np.array([[1.0, 0, 0]]), np.array([[1.0, 0, 0]])],
                                   [np.array([0]), np.array([1])], lambda ids: W[np.asarray(ids)],
                                   keep_intermediates=True)
    assert np.allclose(out2["prob"], 0.5) and out2["idx"][0].tolist() == [0] and out2["idx"][1].tolist() == [1]


def test_perfect_prediction_loss_zero_and_fixed_point():
    C, d = 4, 8
    W = np.zeros((C, d)); W[np.arange(C), np.arange(C)] = 1.0
    cfg = OracleConfig(num_classes=C, dim=d, batch=C, sample_rate=1.0, scale=800.0, margin_type=MARGIN_NONE)
    out = oracle.forward_backward(cfg, [W.copy()], [np.arange(C)], lambda ids: W[np.asarray(ids)])
    assert out["loss"] == pytest.approx(0.0, abs=1e-300)
    assert np.abs(out["grad_x"][0]).max() == 0.0 and np.abs(out["dW"][0]).max() == 0.0


# ---------------------------------------------------------------- library special case (r = 1)
def _torch_dense(x, y, W, s, mt, m, mask=None, ignore_index=None):
    """F.normalize + margin + F.cross_entropy + autograd (library routines) on the dense problem."""
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    cos = torch.nn.functional.normalize(xt, dim=1, eps=1e-12) @ torch.nn.functional.normalize(Wt, dim=1, eps=1e-12).T
    yt = torch.tensor(y)
    oh = torch.nn.functional.one_hot(yt.clamp_min(0), W.shape[0]).bool() & (yt[:, None] >= 0)
    if mt == MARGIN_COSFACE:
        tgt = cos - m
    elif mt == MARGIN_ARCFACE:
        theta = torch.acos(cos.clamp(-1, 1))
        tgt = torch.where(theta + m < math.pi, torch.cos(theta + m), cos - m * math.sin(m))
    else:
        tgt = cos
    logits = s * torch.where(oh, tgt, cos)
    if mask is not None:
        logits = logits.masked_fill(~torch.tensor(mask)[None, :], float("-inf"))
    if ignore_index is None:
        loss = torch.nn.functional.cross_entropy(logits, yt)
    else:
        loss = torch.nn.functional.cross_entropy(logits, yt, ignore_index=ignore_index)
    loss.backward()
    return loss.item(), xt.grad.numpy(), Wt.grad.numpy()


@pytest.mark.parametrize("mt,m", [(MARGIN_ARCFACE, 0.5), (MARGIN_COSFACE, 0.4), (MARGIN_NONE, 0.0)])
@pytest.mark.parametrize("k", [1, 3])
def test_r1_equals_torch_autograd_dense(mt, m, k):
    C, d, B = 37, 16, 5
    W = w_rows_np(4, np.arange(C), d)
    ys = make_labels(2, 0, k, B, C)
    xs = [x.astype(np.float64) for x in make_features(2, 0, k, B, d, labels=ys, dist="trained", sigma=0.3, w_seed=4)]
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=1.0, scale=64.0, margin_type=mt, margin=m)
    out = oracle.forward_backward(cfg, xs, ys, lambda ids: W[np.asarray(ids)])
    L, gx, gW = _torch_dense(np.concatenate(xs), np.concatenate(ys), W, 64.0, mt, m)
    assert out["loss"] == pytest.approx(L, rel=1e-12)
    assert np.allclose(np.concatenate(out["grad_x"]), gx, rtol=1e-9, atol=1e-14)
    assert np.allclose(np.concatenate(out["dW"]), gW, rtol=1e-9, atol=1e-14)


def test_sampled_equals_masked_dense_and_unsampled_rows_get_zero():
    # sampled-mode gradients equal a dense oracle that masks unsampled logits to -inf
    C, d, B, k = 60, 12, 6, 2
    W = w_rows_np(8, np.arange(C), d)
    ys = make_labels(5, 0, k, B, C)
    xs = [x.astype(np.float64) for x in make_features(5, 0, k, B, d)]
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=0.3, scale=64.0,
                       margin_type=MARGIN_ARCFACE, margin=0.5, seed=3)
    out = oracle.forward_backward(cfg, xs, ys, lambda ids: W[np.asarray(ids)], step=7)
    S = np.concatenate(out["idx"])
    mask = np.zeros(C, dtype=bool); mask[S] = True
    L, gx, gW = _torch_dense(np.concatenate(xs), np.concatenate(ys), W, 64.0, MARGIN_ARCFACE, 0.5, mask=mask)
    assert out["loss"] == pytest.approx(L, rel=1e-12)
    assert np.allclose(np.concatenate(out["grad_x"]), gx, rtol=1e-9, atol=1e-14)
    assert np.allclose(np.concatenate(out["dW"]), gW[S], rtol=1e-9, atol=1e-14)
    assert np.abs(gW[~mask]).max() == 0.0


def test_eq9_identity_sampled_prob():
    # P_hat_i = P_i / sum_{j in S} P_j (Eq.9)
    C, d, B = 40, 10, 4
    W = w_rows_np(1, np.arange(C), d)
    ys = make_labels(9, 0, 1, B, C)
    xs = [x.astype(np.float64) for x in make_features(9, 0, 1, B, d)]
    base = dict(num_classes=C, dim=d, batch=B, scale=16.0, margin_type=MARGIN_COSFACE, margin=0.4, seed=2)
    full = oracle.forward_backward(OracleConfig(sample_rate=1.0, **base), xs, ys, lambda i: W[np.asarray(i)], keep_intermediates=True)
    samp = oracle.forward_backward(OracleConfig(sample_rate=0.25, **base), xs, ys, lambda i: W[np.asarray(i)], keep_intermediates=True)
    S = samp["S"]
    P = full["prob"][:, S]
    assert np.allclose(samp["prob"], P / P.sum(axis=1, keepdims=True), rtol=1e-12, atol=1e-300)
    assert np.allclose(samp["prob"].sum(axis=1), 1.0, atol=1e-12)


# ---------------------------------------------------------------- finite differences
@pytest.mark.parametrize("mt,m,r", [(MARGIN_ARCFACE, 0.5, 0.5), (MARGIN_COSFACE, 0.4, 1.0), (MARGIN_NONE, 0.0, 0.3)])
def test_gradients_match_finite_differences(mt, m, r):
    C, d, B, k = 16, 6, 3, 2
    W = w_rows_np(6, np.arange(C), d)
    ys = make_labels(4, 0, k, B, C)
    xs = [x.astype(np.float64) for x in make_features(4, 0, k, B, d, labels=ys, dist="trained", sigma=0.5, w_seed=6)]
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=r, scale=8.0, margin_type=mt, margin=m, seed=1)
    out = oracle.forward_backward(cfg, xs, ys, lambda i: W[np.asarray(i)], step=1)
    h = 1e-6

    def L(xs_, W_):
        return oracle.forward_backward(cfg, xs_, ys, lambda i: W_[np.asarray(i)], step=1)["loss"]

    gx = np.concatenate(out["grad_x"])
    for (rk, n, c) in [(0, 0, 0), (0, 2, 5), (1, 1, 3), (1, 2, 1)]:
        xp = [x.copy() for x in xs]; xm = [x.copy() for x in xs]
        xp[rk][n, c] += h; xm[rk][n, c] -= h
        fd = (L(xp, W) - L(xm, W)) / (2 * h)
        assert fd == pytest.approx(gx[rk * B + n, c], rel=1e-5, abs=1e-9)
    S = np.concatenate(out["idx"])
    gW = np.concatenate(out["dW"])
    for t in [0, len(S) // 2, len(S) - 1]:
        for c in [0, d - 1]:
            Wp = W.copy(); Wm = W.copy()
            Wp[S[t], c] += h; Wm[S[t], c] -= h
            fd = (L(xs, Wp) - L(xs, Wm)) / (2 * h)
            assert fd == pytest.approx(gW[t, c], rel=1e-5, abs=1e-9)


# ---------------------------------------------------------------- invariances
def test_repartition_invariance_at_r1():
    # same global batch, k in {1,2,4} -> identical loss and gradients (Alg.1 is exact)
    C, d, B1 = 50, 8, 8
    W = w_rows_np(3, np.arange(C), d)
    y = make_labels(3, 0, 1, B1, C)[0]
    x = make_features(3, 0, 1, B1, d)[0].astype(np.float64)
    ref = None
    for k in [1, 2, 4]:
        B = B1 // k
        cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=1.0, scale=64.0,
                           margin_type=MARGIN_ARCFACE, margin=0.5)
        out = oracle.forward_backward(cfg, [x[i * B:(i + 1) * B] for i in range(k)],
                                      [y[i * B:(i + 1) * B] for i in range(k)], lambda i: W[np.asarray(i)])
        got = (out["loss"], np.concatenate(out["grad_x"]), np.concatenate(out["dW"]))
        if ref is None:
            ref = got
        else:
            assert got[0] == pytest.approx(ref[0], rel=1e-13)
            assert np.allclose(got[1], ref[1], rtol=1e-11, atol=1e-16)
            assert np.allclose(got[2], ref[2], rtol=1e-11, atol=1e-16)


def test_weight_norm_immaterial():
    # scaling class centres changes nothing but scales dW by 1/alpha
    C, d, B = 30, 8, 5
    W = w_rows_np(2, np.arange(C), d)
    alpha = np.random.default_rng(0).uniform(0.5, 3.0, size=C)
    ys = make_labels(1, 0, 1, B, C)
    xs = [x.astype(np.float64) for x in make_features(1, 0, 1, B, d)]
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=0.5, scale=64.0, margin_type=MARGIN_ARCFACE, margin=0.5)
    a = oracle.forward_backward(cfg, xs, ys, lambda i: W[np.asarray(i)])
    b = oracle.forward_backward(cfg, xs, ys, lambda i: (W * alpha[:, None])[np.asarray(i)])
    assert a["loss"] == pytest.approx(b["loss"], rel=1e-13)
    assert np.allclose(a["grad_x"][0], b["grad_x"][0], rtol=1e-10, atol=1e-16)
    S = a["idx"][0]
    assert np.allclose(a["dW"][0], b["dW"][0] * alpha[S][:, None], rtol=1e-10, atol=1e-16)


def test_init_like_loss_statistical_value():
    # E[L] ~ ln|S| + s^2/(2d) + s sin m for iid directions (SURVEY.md §8(c) smoke value)
    C, d, B = 20000, 512, 64
    ys = make_labels(0, 0, 1, B, C)
    xs = make_features(0, 0, 1, B, d)
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=0.2, scale=64.0, margin_type=MARGIN_ARCFACE, margin=0.5)
    out = oracle.forward_backward(cfg, xs, ys, lambda i: w_rows_np(0, i, d))
    pred = math.log(4000) + 64.0 ** 2 / (2 * d) + 64.0 * math.sin(0.5)
    assert out["loss"] == pytest.approx(pred, rel=0.05)


# ---------------------------------------------------------------- momentum SGD
def test_sgd_reduces_to_vanilla_and_two_step_unroll():
    rng = np.random.default_rng(0)
    W = rng.standard_normal((4, 3)); V = np.zeros((4, 3)); g1 = rng.standard_normal((4, 3)); g2 = rng.standard_normal((4, 3))
    w1, v1 = oracle.sgd_momentum_rows(W, V, g1, lr=0.1, momentum=0.0, weight_decay=0.0)
    assert np.allclose(w1, W - 0.1 * g1, atol=1e-15)
    mu, lam, lr = 0.9, 5e-4, 0.1
    w1, v1 = oracle.sgd_momentum_rows(W, V, g1, lr, mu, lam)
    w2, v2 = oracle.sgd_momentum_rows(w1, v1, g2, lr, mu, lam)
    va = g1 + lam * W
    wa = W - lr * va
    vb = mu * va + g2 + lam * wa
    wb = wa - lr * vb
    assert np.allclose(w2, wb, atol=1e-15) and np.allclose(v2, vb, atol=1e-15)
    w0, v0 = oracle.sgd_momentum_rows(W, V, np.zeros_like(W), lr, mu, 0.0)
    assert np.array_equal(w0, W)                                           # zero-gradient fixed point


def test_sgd_matches_torch_optim_sgd():
    """R15 against the library routine: torch.optim.SGD(momentum=mu, weight_decay=lam, dampening=0, nesterov=False)
    over three steps with fresh gradients (its first step sets the buffer to g + lam w, as the oracle's v = 0
    start does)."""
    rng = np.random.default_rng(3)
    W = rng.standard_normal((5, 7))
    grads = [rng.standard_normal((5, 7)) for _ in range(3)]
    mu, lam, lr = 0.9, 5e-4, 0.07
    p = torch.nn.Parameter(torch.tensor(W, dtype=torch.float64))
    opt = torch.optim.SGD([p], lr=lr, momentum=mu, weight_decay=lam)
    w, v = W.copy(), np.zeros_like(W)
    for g in grads:
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        w, v = oracle.sgd_momentum_rows(w, v, g, lr, mu, lam)
        assert np.allclose(w, p.detach().numpy(), rtol=1e-14, atol=1e-15)
        assert np.allclose(v, opt.state[p]["momentum_buffer"].numpy(), rtol=1e-14, atol=1e-15)


def test_label_out_of_range_is_rejected():
    cfg = OracleConfig(num_classes=10, dim=4, batch=1)
    with pytest.raises(ValueError):
        oracle.forward_backward(cfg, [np.ones((1, 4))], [np.array([10])], lambda i: np.ones((len(i), 4)))


def test_spot_rows_agree_with_full_forward_backward():
    C, d, B, k = 300, 16, 4, 2
    ys = make_labels(2, 0, k, B, C)
    xs = make_features(2, 0, k, B, d)
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=0.1, margin_type=MARGIN_ARCFACE, margin=0.5)
    out = oracle.forward_backward(cfg, xs, ys, lambda i: w_rows_np(0, i, d), step=3)
    S = np.concatenate(out["idx"])
    X = np.concatenate(xs).astype(np.float64); Y = np.concatenate(ys)
    res = oracle.spot_rows(cfg, X, Y, S, lambda i: w_rows_np(0, i, d), [0, 5, 7])
    gx = np.concatenate(out["grad_x"])
    for (lse, lt, g), n in zip(res, [0, 5, 7]):
        assert lse == pytest.approx(out["lse"][n], rel=1e-13)
        assert np.allclose(g, gx[n], rtol=1e-10, atol=1e-16)


def test_spot_cols_agree_with_full_forward_backward():
    C, d, B, k = 400, 16, 5, 2
    ys = make_labels(6, 0, k, B, C)
    xs = make_features(6, 0, k, B, d, labels=ys, dist="trained", sigma=0.3, w_seed=0)
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=0.2, margin_type=MARGIN_ARCFACE, margin=0.5)
    out = oracle.forward_backward(cfg, xs, ys, lambda i: w_rows_np(0, i, d), step=1)
    S = np.concatenate(out["idx"])
    X = np.concatenate(xs).astype(np.float64); Y = np.concatenate(ys)
    cols = [0, 3, len(S) // 2, int(np.searchsorted(S, Y[0]))]
    dW, lse, ct = oracle.spot_cols(cfg, X, Y, S, lambda i: w_rows_np(0, i, d), cols)
    full = np.concatenate(out["dW"])
    assert np.allclose(lse, out["lse"], rtol=1e-13)
    assert np.allclose(ct, out["target_cos"], rtol=1e-13, atol=1e-15)
    assert np.allclose(dW, full[cols], rtol=1e-10, atol=1e-16)


# ---------------------------------------------------------------- method variants
def test_paper_budget_spec_examples():
    # SPEC.md:275-277 (round half up of the paper's product)
    assert oracle.paper_budget(0.1, 1000, 100) == 90
    assert oracle.paper_budget(0.1, 125000, 512) == 12449          # round(12448.8)
    assert oracle.paper_budget(1.0, 500, 37) == 463                 # full complement
    # k = 1, C = 10, labels {2, 5}, r = 0.5 -> 2 positives + round(8 * 0.5) = 4 negatives
    idx, npos = oracle.sample_shard(np.array([2, 5]), 0, 10, 0.5, seed=0, step=0, mode=oracle.SAMPLE_PPRN_PAPER)
    assert npos == 2 and len(idx) == 6 and {2, 5} <= set(idx.tolist())


def test_fully_random_ignores_labels_and_misses_positives():
    # over 1000 trials with C = 100, batch 10, r = 0.1, at least one trial misses a positive
    missed = 0
    counts = np.zeros(100)
    for t in range(1000):
        Y = np.random.default_rng(t).integers(0, 100, size=10)
        idx, npos = oracle.sample_shard(Y, 0, 100, 0.1, seed=3, step=t, mode=oracle.SAMPLE_RANDOM)
        assert npos == 0 and len(idx) == 10
        counts[idx] += 1
        missed += not set(Y.tolist()) <= set(idx.tolist())
    assert missed > 0
    assert np.all(np.abs(counts / 1000 - 0.1) < 0.05)                # uniform over the whole shard


def test_ca_pcc_closed_forms():
    # SPEC.md ca_pcc: every feature equals its centre -> 1.0; features orthogonal to their centres -> 0.0 (Eq.7)
    C, d = 4, 8
    W = np.zeros((C, d)); W[np.arange(C), np.arange(C)] = 1.0
    cfg = OracleConfig(num_classes=C, dim=d, batch=C, sample_rate=1.0, margin_type=MARGIN_NONE)
    out = oracle.forward_backward(cfg, [W.copy()], [np.arange(C)], lambda ids: W[np.asarray(ids)])
    assert out["ca_pcc"] == pytest.approx(1.0, abs=1e-15)
    X = np.zeros((C, d)); X[np.arange(C), np.arange(C) + 4] = 1.0
    out = oracle.forward_backward(cfg, [X], [np.arange(C)], lambda ids: W[np.asarray(ids)])
    assert out["ca_pcc"] == pytest.approx(0.0, abs=1e-15)


@pytest.mark.parametrize("mode", [1, 2])
def test_variants_equal_masked_torch_autograd(mode):
    """PPRN with the paper's budget and fully random sampling against torch autograd of the dense problem with
    unsampled logits masked to -inf; for fully random rows whose positive is unsampled the loss is
    LSE_S - z_t with z_t detached (no positive pull)."""
    C, d, B, k = 80, 12, 6, 2
    W = w_rows_np(2, np.arange(C), d)
    ys = make_labels(8, 0, k, B, C)
    xs = [x.astype(np.float64) for x in make_features(8, 0, k, B, d)]
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=0.2, scale=16.0,
                       margin_type=MARGIN_COSFACE, margin=0.4, seed=5, sample_mode=mode)
    out = oracle.forward_backward(cfg, xs, ys, lambda i: W[np.asarray(i)], step=3)
    S = np.concatenate(out["idx"])
    Y = np.concatenate(ys)
    if mode == 2:
        assert not set(Y.tolist()) <= set(S.tolist())                 # this seed misses some positives
    mask = np.zeros(C, dtype=bool); mask[S] = True
    xt = torch.tensor(np.concatenate(xs), requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    cos = torch.nn.functional.normalize(xt, dim=1) @ torch.nn.functional.normalize(Wt, dim=1).T
    yt = torch.tensor(Y)
    ct = cos[torch.arange(len(Y)), yt]
    zt = 16.0 * (ct - 0.4)
    hit = torch.tensor(mask[Y])
    logits = 16.0 * cos
    logits = torch.where(torch.nn.functional.one_hot(yt, C).bool(), zt[:, None].expand(-1, C), logits)
    logits = logits.masked_fill(~torch.tensor(mask)[None, :], float("-inf"))
    lse = torch.logsumexp(logits, dim=1)
    L = torch.mean(lse - torch.where(hit, zt, zt.detach()))
    L.backward()
    assert out["loss"] == pytest.approx(L.item(), rel=1e-12)
    assert np.allclose(np.concatenate(out["grad_x"]), xt.grad.numpy(), rtol=1e-9, atol=1e-15)
    assert np.allclose(np.concatenate(out["dW"]), Wt.grad.numpy()[S], rtol=1e-9, atol=1e-15)


# ---------------------------------------------------------------- ignore_index = -1 (R28)
@pytest.mark.parametrize("mt,m", [(MARGIN_ARCFACE, 0.5), (MARGIN_COSFACE, 0.4)])
@pytest.mark.parametrize("k", [1, 2])
def test_ignore_index_r1_equals_torch_cross_entropy_ignore_index(mt, m, k):
    """At r = 1 the method is the dense margin softmax: with rows labelled -1 it must equal the library routine
    F.cross_entropy(..., ignore_index=-1) (mean over the other rows) under autograd — loss, grad x and grad W."""
    C, d, B = 41, 16, 6
    W = w_rows_np(4, np.arange(C), d)
    ys = make_labels(5, 0, k, B, C)
    xs = [x.astype(np.float64) for x in make_features(5, 0, k, B, d, labels=ys, dist="trained", sigma=0.3, w_seed=4)]
    ys[0][1] = -1
    ys[-1][4] = -1
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=k, sample_rate=1.0, scale=64.0, margin_type=mt,
                       margin=m, ignore_index=True)
    out = oracle.forward_backward(cfg, xs, ys, lambda ids: W[np.asarray(ids)])
    L, gx, gW = _torch_dense(np.concatenate(xs), np.concatenate(ys), W, 64.0, mt, m, ignore_index=-1)
    assert out["loss"] == pytest.approx(L, rel=1e-12)
    assert np.allclose(np.concatenate(out["grad_x"]), gx, rtol=1e-9, atol=1e-15)
    assert np.allclose(np.concatenate(out["dW"]), gW, rtol=1e-9, atol=1e-15)
    assert not np.any(np.concatenate(out["grad_x"])[[1, k * B - 2]])


def test_ignore_index_equals_dropping_the_rows():
    """Sampled (r < 1): ignoring rows is the same computation as leaving them out of the batch — same sampled ids
    (ignored labels are no positives; the negatives' keys depend only on class ids and the step), same loss,
    same grad_x on the kept rows, zero grad_x on the ignored ones, same class-centre gradients."""
    C, d, B = 3000, 32, 12
    ys = make_labels(7, 0, 1, B, C)
    xs = [x.astype(np.float64) for x in make_features(7, 0, 1, B, d)]
    drop = [2, 3, 9]
    keep = [n for n in range(B) if n not in drop]
    y_ign = ys[0].copy()
    y_ign[drop] = -1
    w = lambda ids: w_rows_np(1, ids, d)
    a = oracle.forward_backward(OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=0.05, seed=3, ignore_index=True),
                                xs, [y_ign], w, step=2)
    b = oracle.forward_backward(OracleConfig(num_classes=C, dim=d, batch=len(keep), sample_rate=0.05, seed=3),
                                [xs[0][keep]], [ys[0][keep]], w, step=2)
    assert np.array_equal(a["idx"][0], b["idx"][0])
    assert a["loss"] == pytest.approx(b["loss"], rel=1e-13)
    assert np.allclose(a["grad_x"][0][keep], b["grad_x"][0], rtol=1e-12, atol=1e-18)
    assert not np.any(a["grad_x"][0][drop])
    assert np.allclose(a["dW"][0], b["dW"][0], rtol=1e-12, atol=1e-18)
    with pytest.raises(ValueError):     # without ignore_index a -1 label is a data error (R7)
        oracle.forward_backward(OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=0.05), xs, [y_ign], w)
