"""Where the end-to-end (host-buffer) step loses time against the device-resident step at C4: device step alone,
with the H2D copies, with the D2H copies, through the async and sync host entries (CUDA events, 20 steps each)."""
import sys
import time
import torch
sys.path.insert(0, ".")
import synth
import paper_2010_05222_b200 as pfc

C, d, B = 10_000_000, 512, 256
layer = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, scale=64.0, margin_type="arcface", margin=0.5,
                      momentum=0.9, weight_decay=5e-4, precision="bf16", seed=1234)
W, V = layer.params()
synth.fill_w_shard(W, 1, 0)
V.zero_()
x = torch.from_numpy(synth.make_features(77, 0, 1, B, d)[0]).cuda()
y = torch.from_numpy(synth.make_labels(77, 0, 1, B, C)[0]).cuda()
xh, yh = x.cpu().pin_memory(), y.cpu().pin_memory()
gx, loss = torch.empty(B, d, device="cuda"), torch.zeros(1, device="cuda")
gh, lh = torch.empty(B, d).pin_memory(), torch.zeros(1).pin_memory()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
K = 20


def timeit(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(K):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / K
    print(f"{name:40s} {e0.elapsed_time(e1) / K:7.4f} ms/step (device)  {wall:7.4f} ms/step (host wall)", flush=True)


timeit("device step", lambda: layer.train_step(x, y, gx, loss, 0.1, s))
timeit("H2D + device step", lambda: (x.copy_(xh, non_blocking=True), y.copy_(yh, non_blocking=True),
                                     layer.train_step(x, y, gx, loss, 0.1, s)))
timeit("device step + D2H", lambda: (layer.train_step(x, y, gx, loss, 0.1, s), gh.copy_(gx, non_blocking=True),
                                     lh.copy_(loss, non_blocking=True)))
timeit("host entry, async", lambda: layer.train_step_host(xh, yh, gh, lh, 0.1, s, sync=False))
timeit("host entry, sync", lambda: layer.train_step_host(xh, yh, gh, lh, 0.1, s))
timeit("device step again", lambda: layer.train_step(x, y, gx, loss, 0.1, s))
