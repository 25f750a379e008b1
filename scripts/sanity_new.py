"""Quick first check of new kernel paths (run under a short `timeout`): one train step each of the all-column
dW+SGD pair kernel (M = 320 / 2048, d = 512 / 256), fp16 logits (fused M = 64 and pair), fused collectives
(loopback-fused and NCCL-fused at world 1), against the float64 oracle."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2010_05222_b200 as pfc  # noqa: E402
from oracle import OracleConfig  # noqa: E402

torch.cuda.set_device(0)


def maxrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def one(C, d, B, comm="nccl", r=0.1):
    t0 = time.time()
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, precision="bf16", seed=3, momentum=0.9,
                      weight_decay=5e-4, comm_mode=comm)
    W, V = L.params()
    synth.fill_w_shard(W, 1, 0)
    V.zero_()
    xs, ys = synth.make_features(5, 0, 1, B, d), synth.make_labels(5, 0, 1, B, C)
    x, y = torch.from_numpy(xs[0]).cuda(), torch.from_numpy(ys[0]).cuda()
    gx, loss = torch.empty_like(x), torch.zeros(1, device="cuda")
    L.train_step(x, y, gx, loss, lr=0.1)
    torch.cuda.synchronize()
    L.check()
    idx = L.sampled()
    cfg = OracleConfig(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type=1, margin=0.5, momentum=0.9,
                       weight_decay=5e-4, seed=3)
    ref = oracle.forward_backward(cfg, xs, ys, lambda i: synth.w_rows_np(1, i, d), step=0)
    w0 = synth.w_rows_np(1, idx, d)
    _, Vr = oracle.sgd_momentum_rows(w0, np.zeros_like(w0), ref["dW"][0], 0.1, 0.9, 5e-4)
    Vg = V[torch.from_numpy(idx).cuda()].cpu().numpy()
    print(f"C={C} d={d} B={B} {comm} flags={L.path_flags()} ids={np.array_equal(idx, ref['idx'][0])} "
          f"loss_rel={abs(loss.item() - ref['loss']) / ref['loss']:.2e} gx={maxrel(gx.cpu().numpy(), ref['grad_x'][0]):.2e} "
          f"V={maxrel(Vg, Vr):.2e} ({time.time() - t0:.1f}s)", flush=True)
    L.close()


for args in [(20000, 512, 320), (20000, 256, 520), (60000, 512, 2048), (3000, 256, 64), (9000, 256, 64, "nccl_fused"),
             (9000, 256, 320, "nccl_fused")]:
    one(*args)
print("SANITY_OK", flush=True)
