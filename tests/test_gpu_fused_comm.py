"""the collectives fused into the kernels (include/pfc.h PFC_COMM_NCCL_FUSED /
PFC_COMM_LOOPBACK_FUSED, csrc/fused_comm.cu). The normalisation kernel stores x_hat and the labels into every rank's
exchange region (Alg.1 L2), the row-combine / prep / finalize kernels exchange the row maxima and
sums through the ranks' slots, reduced in rank order (Alg.1 L6-7), and the dX reduction
stores each owner's rows into the owner's slot, summed in rank order by the x-norm backward (Alg.1 L12-13,
PAPER.md:129-130).

* loopback-fused group vs the plain loopback group (device copies + rank-ascending sums), on one GPU: both reduce in
  rank order, so loss, grad_x, sampled ids and the updated W / V are bit-identical; plus the float64 oracle.
* PFC_COMM_NCCL_FUSED at world size 1: a real NCCL communicator, symmetric window (ncclMemAlloc +
  ncclCommWindowRegister), LSA pointers and device barriers, eager and graph-replayed; equals the plain path."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import OracleConfig

pytestmark = pytest.mark.gpu
pfc = pytest.importorskip("paper_2010_05222_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def group(C, d, B, world, mode, precision="bf16", seed=8, wseed=4):
    layers = []
    for i in range(world):
        L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, margin_type="arcface", margin=0.5,
                          momentum=0.9, weight_decay=5e-4, precision=precision, seed=seed, rank=i, world_size=world,
                          comm_mode=mode)
        W, V = L.params()
        synth.fill_w_shard(W, wseed, L.shard_start)
        V.zero_()
        layers.append(L)
    return layers


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("world,B", [(2, 48), (4, 24), (2, 160), (4, 128)],
                         ids=["w2-fusedM96", "w4-fusedM96", "w2-pairM320", "w4-pairM512"])
@pytest.mark.parametrize("train", [True, False], ids=["train_step", "fwd_bwd"])
def test_loopback_fused_equals_loopback(world, B, precision, train):
    C, d, lr = 30011, 256, 0.1
    plain = group(C, d, B, world, "loopback", precision)
    fused = group(C, d, B, world, "loopback_fused", precision)
    for step in range(2):
        xs = synth.make_features(3, step, world, B, d)
        ys = synth.make_labels(3, step, world, B, C)
        out = []
        for layers in (plain, fused):
            xt = [torch.from_numpy(v).cuda() for v in xs]
            yt = [torch.from_numpy(v).cuda() for v in ys]
            gt = [torch.empty_like(v) for v in xt]
            loss = torch.zeros(1, device="cuda")
            pfc.group_forward_backward(layers, xt, yt, gt, loss, lr=lr if train else None)
            torch.cuda.synchronize()
            for L in layers:
                L.check()
            out.append((loss.item(), [g.cpu().numpy() for g in gt], [L.sampled() for L in layers],
                        None if train else [L.sampled_grad() for L in layers]))
            if not train:
                for L in layers:
                    L.step(lr)
        (la, ga, ia, da), (lb, gb, ib, db) = out
        # bf16: every reduction of both paths runs in a fixed order -> bit-identical. fp32: the SIMT dX / dW
        # contractions accumulate split-K partials with atomics (order not fixed), so compare to rounding level
        exact = precision == "bf16"
        assert (la == lb) if exact else abs(la - lb) <= 1e-6 * abs(la), (la, lb)
        for q in range(world):
            assert np.array_equal(ia[q], ib[q])
            if exact:
                assert np.array_equal(ga[q], gb[q]), (step, q, maxrel(gb[q], ga[q]))
            else:
                assert maxrel(gb[q], ga[q]) <= 1e-5
            if da is not None:
                assert np.array_equal(da[q], db[q]) if exact else maxrel(db[q], da[q]) <= 1e-5
        if step == 0:   # against the float64 oracle (W as initialised)
            cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=world, sample_rate=0.1, margin_type=1,
                               margin=0.5, momentum=0.9, weight_decay=5e-4, seed=8)
            ref = oracle.forward_backward(cfg, xs, ys, lambda ids: synth.w_rows_np(4, ids, d), step=0)
            tl, tg = (1e-3, 2e-2) if precision == "bf16" else (1e-4, 1e-4)
            assert abs(lb - ref["loss"]) / ref["loss"] <= tl
            for q in range(world):
                assert np.array_equal(ib[q], ref["idx"][q])
                assert maxrel(gb[q], ref["grad_x"][q]) <= tg
    for Lp, Lf in zip(plain, fused):
        Wp, Vp = Lp.params()
        Wf, Vf = Lf.params()
        if precision == "bf16":
            assert torch.equal(Wp, Wf) and torch.equal(Vp, Vf)
        else:
            assert maxrel(Vf.cpu(), Vp.cpu()) <= 1e-5
    for L in plain + fused:
        L.close()


@pytest.mark.parametrize("B", [64, 320], ids=["fused-M64", "pair-M320"])
def test_nccl_fused_single_rank_matches_plain(B):
    """The NCCL device-API path on a 1-rank communicator: every kernel stores through the window's LSA address of
    rank 0 and the four LSA barriers run each step; eager, captured and replayed steps equal the plain path."""
    C, d = 9000, 256
    plain = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, precision="bf16", seed=6)
    fused = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, precision="bf16", seed=6,
                          comm_mode="nccl_fused")
    for L in (plain, fused):
        W, V = L.params()
        synth.fill_w_shard(W, 1, 0)
        V.zero_()
    side = torch.cuda.Stream()
    ga, gb = torch.empty(B, d, device="cuda"), torch.empty(B, d, device="cuda")
    la, lb = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    for i in range(4):
        x = torch.from_numpy(synth.make_features(4, i, 1, B, d)[0]).cuda()
        y = torch.from_numpy(synth.make_labels(4, i, 1, B, C)[0]).cuda()
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            plain.train_step(x, y, ga, la, lr=0.1, stream=side)
            fused.train_step(x, y, gb, lb, lr=0.1, stream=side)
        torch.cuda.synchronize()
        fused.check()
        assert la.item() == lb.item()
        assert torch.equal(ga, gb), maxrel(gb.cpu(), ga.cpu())
        assert np.array_equal(plain.sampled(), fused.sampled())
    Wa, Va = plain.params()
    Wb, Vb = fused.params()
    assert torch.equal(Wa, Wb) and torch.equal(Va, Vb)
    plain.close()
    fused.close()
