"""Run a few train steps of one workload (for ncu / compute-sanitizer captures).
    python scripts/prof_step.py [C] [B] [r] [steps] [fused:1|0] [precision]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2010_05222_b200 as pfc

C = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
r = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
fused = (sys.argv[5] != "0") if len(sys.argv) > 5 else True
prec = sys.argv[6] if len(sys.argv) > 6 else "bf16"
d = 512
L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, precision=prec, seed=1, weight_decay=5e-4)
W, V = L.params()
synth.fill_w_shard(W, 1, 0)
V.zero_()
ys = synth.make_labels(0, 0, 1, B, C)
xs = synth.make_features(0, 0, 1, B, d)
x = torch.from_numpy(xs[0]).cuda(); y = torch.from_numpy(ys[0]).cuda()
gx = torch.empty_like(x); loss = torch.zeros(1, device="cuda")
for i in range(steps):
    if fused:
        L.train_step(x, y, gx, loss, lr=0.1)
    else:
        L.forward_backward(x, y, gx, loss)
        L.step(0.1)
torch.cuda.synchronize()
L.check()
print("ok", loss.item(), L.launch_count())
