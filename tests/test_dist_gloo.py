"""Multi-process (gloo, CPU) tests of the N > 1 host logic.

1. The CUDA path's collective decomposition of Alg.1 — all-gather of x_hat and labels, local
   sampled logits with per-shard (max, sum) partials EXCLUDING the target column (R22), all-reduce MAX,
   rescaled all-reduce SUM carrying the target logits, log1p loss, Gc, dX partials, reduce-scatter (R16),
   x-norm backprop — executed rank by rank with real torch.distributed collectives in float64, must reproduce the
   single-process oracle (loss, grad_x, dW, sampled ids).
2. The NCCL unique id made by the library on rank 0 is broadcast intact to every rank (what
   PartialFC.from_process_group does before pfc_init).
3. bench.py's max-over-ranks timing reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _decomposed_rank(rank, world, port, C, d, B, r, mt, m, seed, step, q):
    try:
        _init(rank, world, port)
        import oracle
        import synth
        s = 64.0
        ys = synth.make_labels(4, step, world, B, C)
        xs = synth.make_features(4, step, world, B, d)
        x = torch.tensor(xs[rank], dtype=torch.float64)
        y = torch.tensor(ys[rank])
        # K1 + all-gather (Alg.1 L2)
        xn = x.norm(dim=1)
        xh = x / xn.clamp_min(1e-12)[:, None]
        Xl = [torch.empty_like(xh) for _ in range(world)]
        Yl = [torch.empty_like(y) for _ in range(world)]
        dist.all_gather(Xl, xh)
        dist.all_gather(Yl, y)
        X = torch.cat(Xl).numpy()
        Y = torch.cat(Yl).numpy()
        M = world * B
        # K2-K5 on this shard (the oracle's sampler: bit-exactness of the CUDA sampler is tested on the GPU)
        a, Cl = oracle.shard_range(C, world, rank)
        idx, _ = oracle.sample_shard(Y, a, Cl, r, seed, step)
        Wh, wn = oracle.normalize_rows(synth.w_rows_np(1, idx, d))
        cos = X @ Wh.T
        tcol = np.array([np.searchsorted(idx, yy) if a <= yy < a + Cl else -1 for yy in Y])
        zt_loc = np.zeros(M)
        ct = np.zeros(M)
        for n in range(M):
            if tcol[n] >= 0:
                ct[n] = cos[n, tcol[n]]
                zt_loc[n] = s * oracle.margin_phi(ct[n], mt, m)
        # K6/K7: partials over non-target columns
        Z = s * cos
        mask = np.ones_like(Z, dtype=bool)
        for n in range(M):
            if tcol[n] >= 0:
                mask[n, tcol[n]] = False
        Zm = np.where(mask, Z, -np.inf)
        rowmax = Zm.max(axis=1)
        rowsum = np.where(np.isfinite(rowmax), np.exp(Zm - rowmax[:, None]).sum(axis=1), 0.0)
        # all-reduce MAX, then SUM of rescaled sums + target logits (Alg.1 L6-7)
        gmax = torch.tensor(rowmax)
        dist.all_reduce(gmax, op=dist.ReduceOp.MAX)
        gmax = gmax.numpy()
        red = np.concatenate([np.where(np.isfinite(rowmax), rowsum * np.exp(rowmax - gmax), 0.0), zt_loc])
        red_t = torch.tensor(red)
        dist.all_reduce(red_t)
        red = red_t.numpy()
        S, zt = red[:M], red[M:]
        qv = S * np.exp(gmax - zt)
        loss_n = np.log1p(qv)                 # finalize (R22), valid here since z_t >= max_j z_j or not: use general form
        lse = zt + loss_n
        gt = -qv / (1.0 + qv)
        loss = float(np.mean(loss_n))
        # K8: Gc
        G = s / M * np.exp(Z - lse[:, None])
        for n in range(M):
            if tcol[n] >= 0:
                G[n, tcol[n]] = s / M * gt[n] * oracle.margin_dphi(ct[n], mt, m)
        # K9 + reduce-scatter (Alg.1 L12-13, R16), K10
        dXh = torch.tensor(G @ Wh)
        out = torch.empty(B, d, dtype=torch.float64)
        dist.reduce_scatter(out, list(dXh.chunk(world)))
        dxh = out.numpy()
        xh_np = xh.numpy()
        gx = (dxh - xh_np * np.sum(xh_np * dxh, axis=1, keepdims=True)) / np.maximum(xn.numpy(), 1e-12)[:, None]
        # K11 + norm backprop of W
        dWh = G.T @ X
        dW = (dWh - Wh * np.sum(Wh * dWh, axis=1, keepdims=True)) / np.maximum(wn, 1e-12)[:, None]
        q.put((rank, loss, gx, dW, idx))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, "error", repr(e), None, None))


@pytest.mark.parametrize("world", [2, 3])
def test_collective_decomposition_matches_oracle(world):
    import oracle
    import synth
    C, d, B, r, mt, m, seed, step = 701, 32, 6, 0.2, oracle.MARGIN_ARCFACE, 0.5, 9, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_decomposed_rank, args=(i, world, port, C, d, B, r, mt, m, seed, step, q))
             for i in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rk, loss, gx, dW, idx = q.get(timeout=120)
        assert loss != "error", gx
        res[rk] = (loss, gx, dW, idx)
    for p in procs:
        p.join(timeout=60)
    cfg = oracle.OracleConfig(num_classes=C, dim=d, batch=B, world_size=world, sample_rate=r, margin_type=mt,
                              margin=m, seed=seed)
    ys = synth.make_labels(4, step, world, B, C)
    xs = synth.make_features(4, step, world, B, d)
    ref = oracle.forward_backward(cfg, xs, ys, lambda i: synth.w_rows_np(1, i, d), step=step)
    for rk in range(world):
        loss, gx, dW, idx = res[rk]
        assert loss == pytest.approx(ref["loss"], rel=1e-12)
        assert np.array_equal(idx, ref["idx"][rk])
        assert np.allclose(gx, ref["grad_x"][rk], rtol=1e-9, atol=1e-15)
        assert np.allclose(dW, ref["dW"][rk], rtol=1e-9, atol=1e-15)


def _bcast_rank(rank, world, port, q):
    try:
        _init(rank, world, port)
        import paper_2010_05222_b200 as pfc
        obj = [pfc.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)      # bench.py: ms = max over ranks
        q.put((rank, obj[0], float(t.item())))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error:" + repr(e), 0.0))


def test_unique_id_broadcast_and_max_timing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_rank, args=(i, world, port, q)) for i in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    ids = [g[1] for g in got]
    assert all(isinstance(i, bytes) and len(i) == 128 for i in ids), ids
    assert ids[0] == ids[1]
    assert all(g[2] == float(world) for g in got)
