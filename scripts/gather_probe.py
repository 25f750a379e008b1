"""Probe: HBM bandwidth of random sampled-row reads by access granularity (the W-row pattern of the C4 N=1 step:
1M of 10M rows of 512 fp32, ascending). torch index_select reads [n, w] chunks; chunk widths 2 KB (whole rows),
512 B (dwx d-tiles), 256 B (logits K-blocks). Prints GB/s of bytes read + written."""
import torch

torch.cuda.set_device(0)
C, d, k = 10_000_000, 512, 7812 * 128
W = torch.empty(C, d, device="cuda")
idx = torch.randperm(C, device="cuda")[:k].sort().values


def bench(fn, nbytes, it=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / it / 1e3
    return nbytes / t / 1e9, t * 1e3


for w in (512, 128, 64):
    Wv = W.view(C * (d // w), w)
    per = d // w
    # chunk-major order within 128-row tiles (all chunk c of the tile's rows, then c+1): the fused kernels' order
    tiles = idx.view(-1, 128)
    cidx = (tiles[:, None, :] * per + torch.arange(per, device="cuda")[None, :, None]).reshape(-1)
    out = torch.empty(cidx.numel(), w, device="cuda")
    gbs, ms = bench(lambda: torch.index_select(Wv, 0, cidx, out=out), 2 * cidx.numel() * w * 4)
    print(f"chunk {w * 4:5d} B (tile-chunk-major): {gbs:7.1f} GB/s  {ms:.3f} ms")
    cidx2 = (idx[:, None] * per + torch.arange(per, device="cuda")[None, :]).reshape(-1)
    gbs, ms = bench(lambda: torch.index_select(Wv, 0, cidx2, out=out), 2 * cidx2.numel() * w * 4)
    print(f"chunk {w * 4:5d} B (row-major):        {gbs:7.1f} GB/s  {ms:.3f} ms")
x = torch.empty(k * d, device="cuda")
y = torch.empty_like(x)
gbs, ms = bench(lambda: y.copy_(x), 2 * x.numel() * 4)
print(f"contiguous copy 2 GB:               {gbs:7.1f} GB/s  {ms:.3f} ms")
