import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2010_05222_b200 as pfc
C, d, B, r = 5000, 256, 32, 0.3
def mk():
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, margin_type="cosface", margin=0.4, precision="bf16", seed=3, weight_decay=5e-4)
    W, V = L.params(); synth.fill_w_shard(W, 1, 0); V.zero_(); return L
ys = synth.make_labels(10, 0, 1, B, C); xs = synth.make_features(10, 0, 1, B, d, labels=ys, dist="trained", sigma=0.08, w_seed=1)
x = torch.from_numpy(xs[0]).cuda(); y = torch.from_numpy(ys[0]).cuda(); gx = torch.empty_like(x); loss = torch.zeros(1, device="cuda")
a = mk(); a.forward_backward(x, y, gx, loss); idx = a.sampled(); a.step(0.1); a.check()
b = mk(); b.train_step(x, y, gx, loss, lr=0.1); b.check()
Va = a.params()[1][torch.from_numpy(idx).cuda()].cpu().numpy(); Vb = b.params()[1][torch.from_numpy(idx).cuda()].cpu().numpy()
err = np.abs(Va - Vb).max(axis=1) / np.abs(Va).max()
bad = np.argsort(-err)[:8]
tg = set(ys[0].tolist())
for t in bad: print(t, idx[t], "target" if idx[t] in tg else "neg", err[t], "count", int(np.sum(ys[0] == idx[t])))
print("max err target rows", max(err[t] for t in range(len(idx)) if idx[t] in tg), "non-target", max(err[t] for t in range(len(idx)) if idx[t] not in tg))
