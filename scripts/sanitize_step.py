"""Small workload touching every kernel path once, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck; one tool per run): fused gather + logits and dW+SGD+dX (M <= 256, E-form and softmax-gradient form),
CTA-pair logits + split-K dX + the all-column dW+SGD pair kernel (M > 256), the forward_backward + step path, fp32
SIMT, the loopback-fused collectives, ignore_index and the host-staged shard."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2010_05222_b200 as pfc  # noqa: E402

torch.cuda.set_device(0)


def run(C, d, B, precision="bf16", train=True, steps=2, **kw):
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, precision=precision, seed=1, **kw)
    W, V = L.params()
    if W.is_cuda:
        synth.fill_w_shard(W, 1, 0)
    else:
        W.copy_(synth.w_rows(1, torch.arange(C), d))
    for i in range(steps):
        x = torch.from_numpy(synth.make_features(1, i, 1, B, d)[0]).cuda()
        y = torch.from_numpy(synth.make_labels(1, i, 1, B, C)[0]).cuda()
        if kw.get("ignore_index"):
            y[::5] = -1
        gx, loss = torch.empty_like(x), torch.zeros(1, device="cuda")
        if train:
            L.train_step(x, y, gx, loss, lr=0.1)
        else:
            L.forward_backward(x, y, gx, loss)
            L.step(0.1)
    L.check()
    print(f"ok C={C} d={d} B={B} {precision} train={train} flags={L.path_flags()} loss={loss.item():.4f}", flush=True)
    L.close()


run(3000, 256, 64)                                   # fused M <= 256, E-form
os.environ["PFC_EFORM"] = "0"
run(3000, 256, 64)                                   # fused, softmax-gradient form
del os.environ["PFC_EFORM"]
run(3000, 256, 64, train=False)                      # forward_backward + step
run(6000, 512, 320)                                  # pair logits, split-K dX, all-column dW+SGD
run(6000, 256, 520)
run(3000, 128, 40, precision="fp32")                 # SIMT
run(3000, 256, 64, ignore_index=True)
run(3000, 256, 320, param_location="host")           # staged host shard
layers = [pfc.PartialFC(num_classes=4000, dim=256, batch=24, sample_rate=0.1, seed=2, rank=i, world_size=2,
                        comm_mode="loopback_fused") for i in range(2)]
for Lq in layers:
    synth.fill_w_shard(Lq.params()[0], 1, Lq.shard_start)
xs = [torch.from_numpy(v).cuda() for v in synth.make_features(2, 0, 2, 24, 256)]
ys = [torch.from_numpy(v).cuda() for v in synth.make_labels(2, 0, 2, 24, 4000)]
gs = [torch.empty_like(v) for v in xs]
pfc.group_forward_backward(layers, xs, ys, gs, torch.zeros(1, device="cuda"), lr=0.1)
for Lq in layers:
    Lq.check()
    Lq.close()
print("ok loopback_fused", flush=True)
