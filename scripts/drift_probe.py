"""Does the C4 step time drift as training proceeds (V filling with non-zeros, power)? 10 blocks of 20 device
steps, each with the SM clock, power and throttle reasons sampled by NVML right after the block."""
import sys
import torch
import pynvml
sys.path.insert(0, ".")
import synth
import paper_2010_05222_b200 as pfc

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
C, d, B = 10_000_000, 512, 256
layer = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=0.1, scale=64.0, margin_type="arcface", margin=0.5,
                      momentum=0.9, weight_decay=5e-4, precision="bf16", seed=1234)
W, V = layer.params()
synth.fill_w_shard(W, 1, 0)
V.zero_()
xs = [torch.from_numpy(synth.make_features(77, i, 1, B, d)[0]).cuda() for i in range(4)]
ys = [torch.from_numpy(synth.make_labels(77, i, 1, B, C)[0]).cuda() for i in range(4)]
gx, loss = torch.empty(B, d, device="cuda"), torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
n = 0
for blk in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        layer.train_step(xs[n % 4], ys[n % 4], gx, loss, 0.1, s)
        n += 1
    e1.record(s)
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    torch.cuda.synchronize()
    nz = float((V[:: 1000].abs().sum(1) > 0).float().mean())
    print(f"steps {n:4d}  {e0.elapsed_time(e1) / 20:.4f} ms/step  sm {clk} MHz  {pw:.0f} W  reasons 0x{rs:x}  "
          f"V rows non-zero {nz:.2f}", flush=True)
