#!/usr/bin/env python
"""Partial FC hot-path benchmark (BASELINE.json metric: samples/s of pfc_forward_backward + pfc_step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c2|c3|c3r1|c5]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

One step = one forward+backward of the sampled margin-softmax layer (every SURVEY.md §8(a) row: normalise +
all-gather, PPRN sampling, gather/normalise, logits GEMM + fused margin/LSE partials, global softmax,
softmax gradient, dX and dW GEMMs, reduce-scatter, x-norm backward) plus the lazy momentum-SGD update, on
one synthetic batch already resident in HBM. Default workload (N = 1): BASELINE.json configs[3], 10M
identities, d = 512, B = 256 per GPU, r = 0.1, ArcFace m = 0.5, s = 64, bf16 tensor-core mode; with N GPUs
the 10M classes are sharded over the N ranks (per-GPU batch fixed: "weak").

Prints ONE JSON line on rank 0 (see DESIGN.md §Measurement for every key).
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PFC fwd+bwd samples/s, 10M ids r=0.1, 1/8×B200; tensor-pipe % of peak"
CONFIGS = {
    # name: (C, d, B per GPU, r, margin, m, description)
    "c4": (10_000_000, 512, 256, 0.1, "arcface", 0.5, "10M identities, d=512, B=256/GPU, r=0.1, ArcFace m=0.5 (BASELINE configs[3])"),
    "c1": (1_000, 128, 64, 0.1, "arcface", 0.5, "toy: C=1000, d=128, B=64, r=0.1, ArcFace m=0.5 (BASELINE configs[0]; contract tests)"),
    "c2": (85_742, 512, 128, 0.1, "arcface", 0.5, "MS1MV2-shaped: C=85,742, d=512, B=128/GPU, r=0.1, ArcFace (BASELINE configs[1])"),
    "c3": (360_232, 512, 128, 0.1, "cosface", 0.4, "Glint360K-shaped: C=360,232, d=512, B=128/GPU, r=0.1, CosFace m=0.4 (BASELINE configs[2])"),
    "c3r1": (360_232, 512, 128, 1.0, "cosface", 0.4, "Glint360K-shaped: C=360,232, d=512, B=128/GPU, r=1.0, CosFace m=0.4 (BASELINE configs[2])"),
    "c5": (100_000_000, 512, 256, 0.1, "arcface", 0.5, "100M identities, d=512, B=256/GPU, r=0.1, ArcFace (BASELINE configs[4])"),
    # one rank's exact per-GPU work of the 8-GPU jobs, on one GPU (its C/8 shard and the global batch 8 x 256)
    "c4rank": (1_250_000, 512, 2048, 0.1, "arcface", 0.5, "per-rank proxy of configs[3] on 8 GPUs: 1.25M-class shard, global batch 2048, r=0.1"),
    "c4rank2": (5_000_000, 512, 512, 0.1, "arcface", 0.5, "per-rank proxy of configs[3] on 2 GPUs: 5M-class shard, global batch 512, r=0.1"),
    "c4rank4": (2_500_000, 512, 1024, 0.1, "arcface", 0.5, "per-rank proxy of configs[3] on 4 GPUs: 2.5M-class shard, global batch 1024, r=0.1"),
    "c5rank": (12_500_000, 512, 2048, 0.1, "arcface", 0.5, "per-rank proxy of configs[4] on 8 GPUs: 12.5M-class shard (51 GB W+V), global batch 2048, r=0.1"),
}
SCALE = 64.0
MOMENTUM, WEIGHT_DECAY, LR = 0.9, 5e-4, 0.1


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - only without NVML
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------ roofline
def kernel_work(section, M, k, d):
    """Algorithmic work per launch: (amount, unit, bound) — for the fused kernels
    both the HBM bytes and the flops, as [(amount, unit, bound), ...]; the entry reports the closer roofline."""
    if section in ("logits_gemm", "dx_gemm", "dw_gemm"):
        return [(2.0 * M * k * d, "flop", "tensor")]
    if section == "gather_w":
        return [(4.0 * k * d, "byte", "hbm")]          # read the sampled fp32 rows once
    if section == "gather_logits":                     # fp32 rows once + fp16 cosines out; the logits contraction
        return [(4.0 * k * d + 2.0 * M * k, "byte", "hbm"), (2.0 * M * k * d, "flop", "tensor")]
    if section == "dw_gemm_sgd":                       # W, V read-modify-write of the sampled rows; dW contraction
        return [(16.0 * k * d, "byte", "hbm"), (2.0 * M * k * d, "flop", "tensor")]
    if section == "dwx_sgd":                           # W, V RMW + G' in; dW and dX contractions
        return [(16.0 * k * d + 2.0 * M * k, "byte", "hbm"), (4.0 * M * k * d, "flop", "tensor")]
    if section == "sgd":
        return [(16.0 * k * d, "byte", "hbm")]
    if section == "softmax_grad":
        return [(4.0 * M * k, "byte", "hbm")]          # fp16 cosine in, bf16 gradient out (design minimum)
    if section == "eform_dotw":
        return [(2.0 * M * k, "byte", "hbm")]          # E-form radial dots: the bf16 E entries read once
    return None


def roofline_entry(section, ms, launches, M, k, d, peaks, traffic):
    works = kernel_work(section, M, k, d)
    if works is None or launches == 0:
        return None
    t = ms / launches / 1e3
    cands = []
    for amount, unit, bound in works:
        if bound == "tensor":
            achieved, peak, u, src = amount / t / 1e12, peaks["bf16_tflops_sustained"], "TFLOP/s", "sustained bf16"
        else:
            achieved, peak, u, src = amount / t / 1e9, peaks["hbm_gbs"], "GB/s", "copy"
        cands.append({"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": u,
                      "frac": round(achieved / peak, 4), "per_launch": amount, "peak_src": f"{peaks['src']} ({src})"})
    best = max(cands, key=lambda c: c["frac"])          # the roofline the kernel is closest to
    e = {"kernel": section} | best | {"traffic": traffic.get(section), "avg_ms": round(ms / launches, 4)}
    others = [{kk: c[kk] for kk in ("bound", "achieved", "frac")} for c in cands if c is not best]
    if others:
        e["other_bound"] = others[0]
    return e


# ------------------------------------------------------------------------------------------------ CPU baseline
def cpu_baseline(cfgname, budget_s=25.0, steps=1, warm=0):
    """The oracle (oracle/, float64 numpy, as it stands) on the host cores, on a bounded sample of the
    workload: a contiguous C_ref-class slice of the shard (r, margin, d as the workload), one full oracle step
    (sampler, forward, backward, momentum SGD) with 8 and with 16 samples; the per-step fixed cost and the
    per-sample cost are fitted from the two and extrapolated to the workload's batch B, then scaled by class count
    (every part of the oracle step is proportional to it): samples/s ~ B (C_ref / C) / (t_fix + B t_row)."""
    import torch
    import oracle
    import synth
    from oracle import OracleConfig
    C, d, B, r, mt, m, _ = CONFIGS[cfgname]
    MT = {"none": 0, "arcface": 1, "cosface": 2}

    def one(C_ref, B_ref, step):
        cfg = OracleConfig(num_classes=C_ref, dim=d, batch=B_ref, sample_rate=r, scale=SCALE, margin_type=MT[mt],
                           margin=m, momentum=MOMENTUM, weight_decay=WEIGHT_DECAY, seed=0)
        ys = synth.make_labels(0, step, 1, B_ref, C_ref)
        xs = synth.make_features(0, step, 1, B_ref, d)
        idx, _ = oracle.sample_shard(ys[0], 0, C_ref, r, 0, step)   # untimed: only to pre-generate input rows
        rows = synth.w_rows_np(1, idx, d)
        cache = {"ids": idx, "rows": rows}

        def w_rows(ids):
            ids = np.asarray(ids)
            if ids.shape == cache["ids"].shape and np.array_equal(ids, cache["ids"]):
                return cache["rows"]
            return synth.w_rows_np(1, ids, d)
        t0 = time.perf_counter()
        out = oracle.forward_backward(cfg, xs, ys, w_rows, step=step)
        oracle.sgd_momentum_rows(rows, np.zeros_like(rows), out["dW"][0], LR, MOMENTUM, WEIGHT_DECAY)
        return time.perf_counter() - t0

    probe_c = min(C, 100_000)
    tp = one(probe_c, 8, 0)
    per_class = tp / probe_c
    C_ref = int(min(C, max(20_000, budget_s / (2 * max(steps, 1)) / per_class)))
    t8, t16 = [], []
    for i in range(warm + steps):
        a, b = one(C_ref, 8, 2 * i + 1), one(C_ref, 16, 2 * i + 2)
        if i >= warm:
            t8.append(a)
            t16.append(b)
    a, b = float(np.mean(t8)), float(np.mean(t16))
    t_row = max((b - a) / 8.0, 0.0)
    t_fix = max(a - 8 * t_row, 0.0)
    t_step = t_fix + B * t_row
    value = B * (C_ref / C) / t_step
    return {"value": value, "unit": "samples/s", "cores": torch.get_num_threads(), "kind": "oracle",
            "sample": f"oracle steps on a {C_ref}-class slice of the {C}-class shard (r={r}, d={d}) with 8 and 16 "
                      f"samples ({a:.3f} s, {b:.3f} s per full step: sampler, fwd, bwd, SGD, float64 numpy); fitted "
                      f"{t_fix:.3f} s/step + {t_row*1e3:.1f} ms/sample, extrapolated to B={B} and scaled by class "
                      f"count C/C_ref; {len(t8)} step pair(s)",
            "seconds_per_step": t_step * C / C_ref}


# ------------------------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--params", default="device", choices=["device", "host"],
                    help="where W and V live: HBM (default) or page-locked host memory (capacity mode, f4)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    C, d, B, r, mt, m, desc = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        budget = max(30.0, 150.0 / max(1, args.steps + args.warmup)) * (args.steps + args.warmup)
        cb = cpu_baseline(args.config, budget_s=min(budget, 150.0), steps=args.steps, warm=args.warmup)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["seconds_per_step"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "oracle": "oracle/pfc.py (float64 numpy, CPU)"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    import synth
    import paper_2010_05222_b200 as pfc

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    layer = pfc.PartialFC.from_process_group(**dict(
        num_classes=C, dim=d, batch=B, sample_rate=r, scale=SCALE, margin_type=mt, margin=m, momentum=MOMENTUM,
        weight_decay=WEIGHT_DECAY, precision=args.precision, seed=1234, device=local,
        param_location=args.params)) if world > 1 else \
        pfc.PartialFC(num_classes=C, dim=d, batch=B, sample_rate=r, scale=SCALE, margin_type=mt, margin=m,
                      momentum=MOMENTUM, weight_decay=WEIGHT_DECAY, precision=args.precision, seed=1234, device=local,
                      param_location=args.params)
    W, V = layer.params()
    if args.params == "host":       # page-locked host shard: rows generated on the GPU, copied
        tmp = torch.empty(1 << 18, d, device="cuda")
        for r0 in range(0, layer.shard_size, tmp.shape[0]):
            n = min(tmp.shape[0], layer.shard_size - r0)
            synth.fill_w_shard(tmp[:n], 1, layer.shard_start + r0)
            W[r0:r0 + n].copy_(tmp[:n])
        del tmp
    else:
        synth.fill_w_shard(W, 1, layer.shard_start)
    V.zero_()
    M, k = layer.global_batch, layer.k_max
    # synthetic init-like batches, resident in HBM before the timed region
    NB = 4
    xs, ys = [], []
    for i in range(NB):
        yl = synth.make_labels(77, i, world, B, C)[rank]
        xl = synth.make_features(77, i, world, B, d)[rank]
        xs.append(torch.from_numpy(xl).cuda())
        ys.append(torch.from_numpy(yl).cuda())
    gx = torch.empty(B, d, device="cuda")
    loss = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()          # a capturable stream: the library replays the step as a CUDA graph
    torch.cuda.set_stream(stream)

    def step(i):
        layer.train_step(xs[i % NB], ys[i % NB], gx, loss, LR, stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    layer.check()

    # ---------------- timed region (device-resident inputs; the step is replayed as a CUDA graph)
    l0 = layer.launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = layer.launch_count() - l0
    loss_val = float(loss.item())
    layer.check()
    t = torch.tensor([ms_total], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = M * args.steps / (ms_max / 1e3)

    # ---------------- per-kernel times: the same K steps again with CUDA events between the kernels (eager
    # launches on the same stream: event records are not replayable per step inside one graph)
    layer.profile(True)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for i in range(args.steps):
        step(i)
    p1.record(stream)
    prof = layer.profile_read()
    layer.profile(False)
    ms_prof = p0.elapsed_time(p1)
    # section names by the kernel path (include/pfc.h PFC_PATH_*): the train step fuses the momentum-SGD update
    # into the dW contraction (section 8; sgd 9 empty); with the fused gather the logits section holds
    # gather + logits (section 2 keeps the target cosines); with the fused dW/dX kernel section 6 holds
    # dW + SGD + dX and section 8 is empty
    flags = layer.path_flags()
    rename = {"dw_gemm": "dw_gemm_sgd"}
    if flags & layer.PATH_FUSED_GATHER:
        rename |= {"logits_gemm": "gather_logits", "gather_w": "target_cos"}
    if flags & layer.PATH_FUSED_DWX:
        rename |= {"dx_gemm": "dwx_sgd"}
    if flags & layer.PATH_EFORM:                 # E-form: no softmax-gradient pass; section 5 = per-row preparation
        # (+ the radial-dot pass over E when dX is not fused into the dW kernel)
        rename |= {"softmax_grad": "eform_prep" if flags & layer.PATH_FUSED_DWX else "eform_dotw"}
    prof = {rename.get(s, s): v for s, v in prof.items()}
    if flags & layer.PATH_FUSED_DWX:
        prof.pop("dw_gemm_sgd", None)        # empty: dW + SGD ran inside dwx_sgd

    # ---------------- end-to-end through the C-ABI with host buffers (pinned), copies inside the timed region
    xh = [x.cpu().pin_memory() for x in xs]
    yh = [y.cpu().pin_memory() for y in ys]
    gh = torch.empty(B, d).pin_memory()
    lh = torch.zeros(1).pin_memory()
    for i in range(2):
        layer.train_step_host(xh[i % NB], yh[i % NB], gh, lh, LR, stream)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        layer.train_step_host(xh[i % NB], yh[i % NB], gh, lh, LR, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    te = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = M * args.steps / (float(te.item()) / 1e3)

    if rank == 0:
        peaks = load_peaks()
        traffic = {}
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            tj = json.load(open(tp)).get("workloads", {}).get(f"{args.config}/{world}", {})
            traffic = tj.get("bytes_per_launch", {})
        entries = [e for e in (roofline_entry(s, ms, n, M, k, d, peaks, traffic) for s, (ms, n) in prof.items()) if e]
        gemm = [prof[s_] for s_ in ("logits_gemm", "gather_logits", "dx_gemm", "dwx_sgd", "dw_gemm_sgd")
                if s_ in prof and prof[s_][1]]
        gemm_ms = sum(ms / n for ms, n in gemm)
        gemm_tensor_frac = (3 * 2.0 * M * k * d / (gemm_ms / 1e3) / 1e12 / peaks["bf16_tflops_sustained"]
                            if gemm_ms else None)
        dominant = max(prof.items(), key=lambda kv: kv[1][0])[0]
        dom = next((e for e in entries if e["kernel"] == dominant), None)
        if dom is None and entries:
            dom = max(entries, key=lambda e: e["avg_ms"])
        sections = {s: {"ms_per_step": round(ms / args.steps, 4), "share": round(ms / ms_prof, 4)}
                    for s, (ms, n) in prof.items() if n}
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": desc, "num_classes": C, "dim": d, "batch_per_gpu": B, "global_batch": M,
                       "sample_rate": r, "k_per_gpu": k, "shard_rows": layer.shard_size, "margin": f"{mt} {m}",
                       "scale": SCALE, "parallelism": f"class-parallel x{world}", "params": args.params,
                       "l2": "inputs larger than L2 (W+V shard %.1f GB, %.1f GB of sampled rows per step)"
                             % (2 * layer.shard_size * d * 4 / 1e9, k * d * 4 / 1e9)},
            "clocks": clk.summary(),
            "e2e": {"value": round(e2e_value, 1), "unit": "samples/s", "h2d_bytes_per_step": B * d * 4 + B * 8,
                    "d2h_bytes_per_step": B * d * 4 + 4},
            "gpu_launches": launches,
            "roofline": {kk: dom[kk] for kk in ("bound", "achieved", "peak", "unit", "frac", "traffic")} | {
                "kernel": dom["kernel"], "peak_src": dom["peak_src"]} if dom else None,
            "kernels": entries, "sections": sections, "loss": loss_val,
            "gemm_tensor_frac": round(gemm_tensor_frac, 4) if gemm_tensor_frac else None,
            "gemm_tensor_frac_note": "the three contractions' 6 M k d flops / the summed event time of the kernels holding them / bf16 "
                                     "peak (the metric's tensor-pipe share; at N = 1 the fused dW kernel is HBM-bound)",
            "step_ms_rank0": round(ms_total / args.steps, 4),
            "step_ms_eager_profiled": round(ms_prof / args.steps, 4),
            "kernel_timing": "CUDA events between the kernels on the launching stream, same K steps run eagerly "
                             "right after the graph-replayed timed region",
        }
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(args.config, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {kk: cb[kk] for kk in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
