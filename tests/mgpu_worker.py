"""Worker of tests/test_multigpu.py (launched by torchrun, one process per GPU, NCCL): runs the N-rank fused train
step of paper_2010_05222_b200 over a real NCCL communicator (eager first call, then captured and graph-replayed),
gathers every rank's outputs to rank 0, and there checks them against (a) the loopback group — all N ranks in one
process on one GPU, the same kernels with device-copy collectives — and (b) the float64 oracle."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2010_05222_b200 as pfc  # noqa: E402
from oracle import OracleConfig  # noqa: E402


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def main():
    C, d, B, r, lr, steps = int(sys.argv[1]), 512, int(sys.argv[2]), 0.1, 0.1, 3
    comm = sys.argv[3] if len(sys.argv) > 3 else "nccl"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kw = dict(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type="arcface", margin=0.5, momentum=0.9,
              weight_decay=5e-4, precision="bf16", seed=21)
    L = pfc.PartialFC.from_process_group(device=local, comm_mode=comm, **kw)
    W, V = L.params()
    synth.fill_w_shard(W, 3, L.shard_start)
    V.zero_()
    side = torch.cuda.Stream()
    x = torch.empty(B, d, device="cuda")
    y = torch.empty(B, dtype=torch.int64, device="cuda")
    gx, loss = torch.empty(B, d, device="cuda"), torch.zeros(1, device="cuda")
    outs = []
    for i in range(steps):   # call 1 eager, call 2 captured, call 3 replayed
        x.copy_(torch.from_numpy(synth.make_features(30, i, world, B, d)[rank]))
        y.copy_(torch.from_numpy(synth.make_labels(30, i, world, B, C)[rank]))
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            L.train_step(x, y, gx, loss, lr=lr, stream=side)
        torch.cuda.synchronize()
        L.check()
        outs.append({"loss": loss.item(), "gx": gx.cpu().numpy(), "idx": L.sampled()})
    idx_last = outs[-1]["idx"]
    loc = torch.from_numpy(idx_last - L.shard_start).cuda()
    mine = {"outs": outs, "W": W[loc].cpu().numpy(), "V": V[loc].cpu().numpy(), "start": L.shard_start,
            "flags": L.path_flags()}
    allr = [None] * world
    dist.gather_object(mine, allr if rank == 0 else None, dst=0)
    L.close()
    if rank == 0:
        report = check(allr, C, d, B, r, lr, steps, world, kw, comm)
        print("MGPU_REPORT " + json.dumps(report), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def check(allr, C, d, B, r, lr, steps, world, kw, comm):
    # (a) the loopback group on this GPU: the same N ranks, same inputs, collectives as device copies / sums (or, for
    # the fused NCCL path, the same fused kernels storing into the other contexts' regions)
    lb = "loopback_fused" if comm == "nccl_fused" else "loopback"
    layers = [pfc.PartialFC(rank=i, world_size=world, comm_mode=lb, device=0, **kw) for i in range(world)]
    for Lq in layers:
        Wq, Vq = Lq.params()
        synth.fill_w_shard(Wq, 3, Lq.shard_start)
        Vq.zero_()
    # a + b is order-free: NCCL and the loopback sums agree bit for bit at N = 2; the fused path reduces in rank
    # order on every rank, exactly like its loopback group, at any N
    exact = world == 2 or comm == "nccl_fused"
    rep = {"world": world, "comm": comm, "exact_expected": exact, "steps": []}
    for i in range(steps):
        xs = synth.make_features(30, i, world, B, d)
        ys = synth.make_labels(30, i, world, B, C)
        xt = [torch.from_numpy(v).cuda() for v in xs]
        yt = [torch.from_numpy(v).cuda() for v in ys]
        gt = [torch.empty(B, d, device="cuda") for _ in range(world)]
        lo = torch.zeros(1, device="cuda")
        pfc.group_forward_backward(layers, xt, yt, gt, lo, lr=lr)
        torch.cuda.synchronize()
        st = {"loss_nccl": allr[0]["outs"][i]["loss"], "loss_loopback": lo.item()}
        for q in range(world):
            o = allr[q]["outs"][i]
            assert np.array_equal(o["idx"], layers[q].sampled()), ("ids differ from loopback", i, q)
            st[f"gx_vs_loopback_r{q}"] = maxrel(o["gx"], gt[q].cpu().numpy())
            if exact:
                assert np.array_equal(o["gx"], gt[q].cpu().numpy()), ("grad_x not bit-identical", i, q)
        if exact:
            assert st["loss_nccl"] == st["loss_loopback"], st
        else:
            assert abs(st["loss_nccl"] - st["loss_loopback"]) <= 1e-6 * abs(st["loss_loopback"]), st
            assert max(v for k, v in st.items() if k.startswith("gx_vs")) <= 1e-5, st
        rep["steps"].append(st)
    for q in range(world):
        Wq, Vq = layers[q].params()
        loc = torch.from_numpy(allr[q]["outs"][-1]["idx"] - layers[q].shard_start).cuda()
        wl, vl = Wq[loc].cpu().numpy(), Vq[loc].cpu().numpy()
        rep[f"V_vs_loopback_r{q}"] = maxrel(allr[q]["V"], vl)
        if exact:
            assert np.array_equal(allr[q]["V"], vl) and np.array_equal(allr[q]["W"], wl), ("W/V not bit-identical", q)
        else:
            assert rep[f"V_vs_loopback_r{q}"] <= 1e-5
    for Lq in layers:
        Lq.close()
    # (b) the float64 oracle on the first step (W as initialised): ids bit-exact, north-star bf16 bars
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, world_size=world, sample_rate=r, margin_type=1, margin=0.5,
                       momentum=0.9, weight_decay=5e-4, seed=21)
    xs, ys = synth.make_features(30, 0, world, B, d), synth.make_labels(30, 0, world, B, C)
    ref = oracle.forward_backward(cfg, xs, ys, lambda ids: synth.w_rows_np(3, ids, d), step=0)
    rep["oracle_loss_rel"] = abs(allr[0]["outs"][0]["loss"] - ref["loss"]) / ref["loss"]
    rep["oracle_gx"] = max(maxrel(allr[q]["outs"][0]["gx"], ref["grad_x"][q]) for q in range(world))
    for q in range(world):
        assert np.array_equal(allr[q]["outs"][0]["idx"], ref["idx"][q]), ("ids differ from the oracle", q)
    assert rep["oracle_loss_rel"] <= 1e-3 and rep["oracle_gx"] <= 2e-2, rep
    rep["ok"] = True
    return rep


if __name__ == "__main__":
    main()
