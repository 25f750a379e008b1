"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (bf16 tensor-core mode,
fused train step where the whole step is compared).

* C2 MS1MV2-shaped (C = 85,742, d = 512, B = 128/GPU, r = 0.1, ArcFace) on 8 ranks and C3 Glint360K-shaped
  (C = 360,232, CosFace 0.4, r = 0.1 on 8 ranks; r = 1.0 on 1 rank): every rank simulated on the one GPU
  (loopback group), compared element by element with the oracle (ids bit-exact; loss, grad_x, updated V rows).
* C4 10M identities on one GPU (the bench workload: C_local = 10M, k = 1M, M = 256): sampled ids bit-exact over
  the whole 10M-class shard; per-row log-sum-exp, loss terms and grad_x on sampled rows; dW on sampled classes
  (oracle.spot_rows / spot_cols compute those one by one).
Tolerances: the north-star bf16 bars (1e-3 relative loss, 2e-2 max-relative gradients; R19)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import OracleConfig

pytestmark = pytest.mark.gpu
pfc = pytest.importorskip("paper_2010_05222_b200")
MT = {"none": 0, "arcface": 1, "cosface": 2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def maxrel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("C,world,B,r,mt,m", [
    (85_742, 8, 128, 0.1, "arcface", 0.5),     # BASELINE configs[1]
    (85_742, 8, 256, 0.1, "arcface", 0.5),     # configs[1] shape at M = 2048: logits and dW + SGD on CTA pairs
    (360_232, 8, 128, 0.1, "cosface", 0.4),    # configs[2], r = 0.1
    (360_232, 1, 128, 1.0, "cosface", 0.4),    # configs[2], r = 1.0 (full softmax over 360k classes)
])
def test_group_train_step_full_size(C, world, B, r, mt, m):
    d, lr, wseed, seed = 512, 0.1, 3, 17
    layers = []
    for i in range(world):
        L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type=mt, margin=m, momentum=0.9,
                          weight_decay=5e-4, precision="bf16", seed=seed, rank=i, world_size=world,
                          comm_mode="loopback")
        W, V = L.params()
        synth.fill_w_shard(W, wseed, L.shard_start)
        V.zero_()
        layers.append(L)
    ys = synth.make_labels(21, 0, world, B, C)
    xs = synth.make_features(21, 0, world, B, d)
    xt = [torch.from_numpy(x).cuda() for x in xs]
    yt = [torch.from_numpy(y).cuda() for y in ys]
    gt = [torch.empty_like(x) for x in xt]
    loss = torch.zeros(1, device="cuda")
    if world == 1:
        layers[0].train_step(xt[0], yt[0], gt[0], loss, lr=lr)
    else:
        pfc.group_forward_backward(layers, xt, yt, gt, loss, lr=lr)
    torch.cuda.synchronize()
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=world, sample_rate=r, margin_type=MT[mt], margin=m,
                       momentum=0.9, weight_decay=5e-4, seed=seed)
    ref = oracle.forward_backward(cfg, xs, ys, lambda i: synth.w_rows_np(wseed, i, d), step=0)
    assert abs(loss.item() - ref["loss"]) / ref["loss"] <= 1e-3
    for i, L in enumerate(layers):
        idx = L.sampled()
        assert np.array_equal(idx, ref["idx"][i])
        assert maxrel(gt[i].cpu().numpy(), ref["grad_x"][i]) <= 2e-2
        W, V = L.params()
        loc = torch.from_numpy(idx - L.shard_start).cuda()
        w0 = synth.w_rows_np(wseed, idx, d)
        Wr, Vr = oracle.sgd_momentum_rows(w0, np.zeros_like(w0), ref["dW"][i], lr, 0.9, 5e-4)
        assert maxrel(V[loc].cpu().numpy(), Vr) <= 2e-2
        assert maxrel(W[loc].cpu().numpy(), Wr) <= 1e-5
    for L in layers:
        L.close()


def test_c4_ten_million_ids_one_gpu_sampled_outputs():
    C, d, B, r, m, seed, wseed = 10_000_000, 512, 256, 0.1, 0.5, 1234, 1
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type="arcface", margin=m, momentum=0.9,
                      weight_decay=5e-4, precision="bf16", seed=seed)
    W, V = L.params()
    synth.fill_w_shard(W, wseed, 0)
    V.zero_()
    ys = synth.make_labels(77, 0, 1, B, C)
    xs = synth.make_features(77, 0, 1, B, d)
    x = torch.from_numpy(xs[0]).cuda()
    y = torch.from_numpy(ys[0]).cuda()
    gx = torch.empty_like(x)
    loss = torch.zeros(1, device="cuda")
    L.forward_backward(x, y, gx, loss)
    idx = L.sampled()
    lse = L.lse()
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type=oracle.MARGIN_ARCFACE, margin=m,
                       seed=seed)
    ref_idx, _ = oracle.sample_shard(ys[0], 0, C, r, seed, 0)
    assert len(idx) == 1_000_000 and np.array_equal(idx, ref_idx)        # bit-exact over the 10M-class shard
    S = ref_idx
    Wrows = synth.w_rows_np(wseed, S, d)

    def w_rows(ids):
        ids = np.asarray(ids)
        return Wrows if ids.shape == S.shape and ids[0] == S[0] and ids[-1] == S[-1] else synth.w_rows_np(wseed, ids, d)

    X = xs[0].astype(np.float64)
    Y = ys[0]
    rows = [0, 17, 101, 255]
    gx_h = gx.cpu().numpy()
    for (lse_r, lt, g), n in zip(oracle.spot_rows(cfg, X, Y, S, w_rows, rows), rows):
        assert abs(lse[n] - lse_r) / abs(lse_r) <= 1e-3 * 0.1     # log-sum-exp ~ 48: well inside the loss bar
        assert maxrel(gx_h[n], g) <= 2e-2
    cols = sorted(set([0, 1, 500_000, 999_999] + [int(np.searchsorted(S, Y[n])) for n in rows]))
    dW_ref, lse_all, ct_all = oracle.spot_cols(cfg, X, Y, S, w_rows, cols)
    loss_ref = float(np.mean(lse_all - 64.0 * oracle.margin_phi(ct_all, oracle.MARGIN_ARCFACE, m)))
    assert abs(loss.item() - loss_ref) / loss_ref <= 1e-3
    dW = L.sampled_grad()
    assert maxrel(dW[cols], dW_ref) <= 2e-2
    # the lazy update touches exactly the sampled rows
    W_before = W[torch.from_numpy(S[:1000]).cuda()].clone()
    L.step(0.1)
    L.check()
    W_after = W[torch.from_numpy(S[:1000]).cuda()]
    V_rows = V[torch.from_numpy(S[cols]).cuda()].cpu().numpy()
    _, Vr = oracle.sgd_momentum_rows(Wrows[cols], np.zeros((len(cols), d)), dW_ref, 0.1, 0.9, 5e-4)
    assert maxrel(V_rows, Vr) <= 2e-2
    assert not torch.equal(W_before, W_after)
    L.close()


def _w_rows_chunked(wseed, ids, d, chunk=1 << 16):
    ids = np.asarray(ids)
    return np.concatenate([synth.w_rows_np(wseed, ids[i:i + chunk], d) for i in range(0, len(ids), chunk)])


def test_c5_per_rank_shape_spot_parity():
    """BASELINE configs[4] (100M identities over 8 B200) at one rank's exact shape: a 12.5M-class shard (51 GB of
    W + V in HBM), M = 2048 (the all-gathered batch of 8 x 256), k = 1.25M, the bf16 E-form train step the bench
    times (CTA-pair logits and dW + SGD; E has 2.56e9 > 2^31 entries). Sampled ids bit-exact over the whole
    shard; the loss over all 2048 rows; grad_x on spot rows (oracle.spot_rows); the updated V and W of spot
    sampled classes (V = dW + lambda w from zero momentum; oracle.spot_cols) — all at the north-star bars."""
    import _parity
    C, d, B, r, m, seed, wseed, lr, lam = 12_500_000, 512, 2048, 0.1, 0.5, 77, 2, 0.1, 5e-4
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type="arcface", margin=m, momentum=0.9,
                      weight_decay=lam, precision="bf16", seed=seed)
    assert L.path_flags() == 9      # CTA-pair kernels, E-form
    W, V = L.params()
    synth.fill_w_shard(W, wseed, 0)
    V.zero_()
    ys = synth.make_labels(91, 0, 1, B, C)
    xs = synth.make_features(91, 0, 1, B, d)
    x, y = torch.from_numpy(xs[0]).cuda(), torch.from_numpy(ys[0]).cuda()
    gx, loss = torch.empty_like(x), torch.zeros(1, device="cuda")
    L.train_step(x, y, gx, loss, lr=lr)
    torch.cuda.synchronize()
    L.check()
    idx = L.sampled()
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type=oracle.MARGIN_ARCFACE, margin=m,
                       weight_decay=lam, seed=seed)
    S, _ = oracle.sample_shard(ys[0], 0, C, r, seed, 0)
    assert len(S) == 1_250_000 and np.array_equal(idx, S)        # bit-exact over the 12.5M-class shard
    Wrows = _w_rows_chunked(wseed, S, d)

    def w_rows(ids):
        ids = np.asarray(ids)
        return Wrows if ids.shape == S.shape and ids[0] == S[0] and ids[-1] == S[-1] else synth.w_rows_np(wseed, ids, d)

    X, Y = xs[0].astype(np.float64), ys[0]
    rows = [0, 1, 777, 1500, 2047]
    cols = sorted(set([0, 1, 625_000, 1_249_999] + [int(np.searchsorted(S, Y[n])) for n in rows[:3]]))
    dW_ref, lse_all, ct_all = oracle.spot_cols(cfg, X, Y, S, w_rows, cols)
    loss_ref = float(np.mean(lse_all - 64.0 * oracle.margin_phi(ct_all, oracle.MARGIN_ARCFACE, m)))
    gx_h = gx.cpu().numpy()
    gx_err = max(maxrel(gx_h[n], g) for (_, _, g), n in zip(oracle.spot_rows(cfg, X, Y, S, w_rows, rows), rows))
    _, Vr = oracle.sgd_momentum_rows(Wrows[cols], np.zeros((len(cols), d)), dW_ref, lr, 0.9, lam)
    Wr = Wrows[cols] - lr * Vr
    loc = torch.from_numpy(S[cols]).cuda()
    v_err = maxrel(V[loc].cpu().numpy(), Vr)
    w_err = maxrel(W[loc].cpu().numpy(), Wr)
    errs = _parity.record("test_c5_per_rank_shape_spot_parity", "bf16", loss_rel=abs(loss.item() - loss_ref) / loss_ref,
                          grad_x=gx_err, V=v_err, W=w_err, L=loss_ref)
    assert errs["loss_rel"] <= 1e-3 and gx_err <= 2e-2 and v_err <= 2e-2, errs
    assert w_err <= 1e-6 + lr * 2e-2 * np.max(np.abs(Vr)) / np.max(np.abs(Wr)), errs
    L.close()
