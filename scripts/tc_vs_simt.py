"""Diagnostic: run one forward/backward with the tcgen05 GEMMs and with the FFMA GEMMs (PFC_GEMM=simt) on the
same inputs and compare loss, LSE, grad_x and dW (localises a wrong contraction)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2010_05222_b200 as pfc


def run(C, d, B, r, backend):
    if backend == "simt":
        os.environ["PFC_GEMM"] = "simt"
    else:
        os.environ.pop("PFC_GEMM", None)
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, precision="bf16", seed=3)
    W, V = L.params()
    synth.fill_w_shard(W, 1, 0)
    ys = synth.make_labels(1, 0, 1, B, C)
    xs = synth.make_features(1, 0, 1, B, d)
    x = torch.from_numpy(xs[0]).cuda(); y = torch.from_numpy(ys[0]).cuda()
    gx = torch.empty_like(x); loss = torch.zeros(1, device="cuda")
    L.forward_backward(x, y, gx, loss)
    L.check()
    out = dict(loss=loss.item(), lse=L.lse(), gx=gx.cpu().numpy(), dW=L.sampled_grad(), idx=L.sampled())
    L.close()
    return out


for (C, d, B, r) in [(1000, 128, 64, 0.1), (20000, 512, 96, 0.05), (100000, 512, 256, 0.1), (50000, 512, 300, 0.3)]:
    a = run(C, d, B, r, "tc")
    b = run(C, d, B, r, "simt")
    rel = lambda u, v: float(np.max(np.abs(u - v)) / max(np.max(np.abs(v)), 1e-30))
    print(f"C={C} d={d} B={B} r={r}: idx_eq={np.array_equal(a['idx'], b['idx'])} loss {a['loss']:.6f} vs {b['loss']:.6f} "
          f"lse {rel(a['lse'], b['lse']):.2e} gx {rel(a['gx'], b['gx']):.2e} dW {rel(a['dW'], b['dW']):.2e}", flush=True)
