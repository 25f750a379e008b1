"""Per-rank step time of a K-GPU job, emulated on one GPU (T_solo of DESIGN.md §7): the K ranks of the job are
loopback contexts driven by pfc_group_train_step; one group step runs every rank's kernels back to back, so the
per-rank time is the group time / K (collectives are device copies/sums here, NCCL on real GPUs).
    python scripts/bench_emulate.py [--world 8] [--config c4] [--steps 10] [--warmup 3]"""
import argparse, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
import paper_2010_05222_b200 as pfc
from bench import CONFIGS, SCALE, MOMENTUM, WEIGHT_DECAY, LR

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
C, d, B, r, mt, m, desc = CONFIGS[a.config]
K = a.world
layers = []
for i in range(K):
    L = pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, scale=SCALE, margin_type=mt, margin=m,
                      momentum=MOMENTUM, weight_decay=WEIGHT_DECAY, precision="bf16", seed=1234, rank=i, world_size=K,
                      comm_mode="loopback")
    W, V = L.params()
    synth.fill_w_shard(W, 1, L.shard_start)
    V.zero_()
    layers.append(L)
ys = synth.make_labels(77, 0, K, B, C)
xs = synth.make_features(77, 0, K, B, d)
xt = [torch.from_numpy(x).cuda() for x in xs]
yt = [torch.from_numpy(y).cuda() for y in ys]
gt = [torch.empty_like(x) for x in xt]
loss = torch.zeros(1, device="cuda")
for _ in range(a.warmup):
    pfc.group_forward_backward(layers, xt, yt, gt, loss, lr=LR)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    pfc.group_forward_backward(layers, xt, yt, gt, loss, lr=LR)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
per_rank = ms / K
M = K * B
k = layers[0].k_max
print(json.dumps({"workload": desc, "emulated_world": K, "group_step_ms": round(ms, 4), "per_rank_step_ms": round(per_rank, 4),
                  "projected_samples_per_s": round(M / (per_rank / 1e3), 1), "M": M, "k_per_rank": k,
                  "gemm_tflops_per_rank": round(6 * M * k * d / (per_rank / 1e3) / 1e12, 1), "loss": loss.item()}))
