"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only produces inputs (class-centre matrix W,
features x, labels y) shaped like the paper's workloads. Both the oracle and the
CUDA path consume exactly the same values:

* W rows are a counter-based integer hash of (seed, row, column) evaluated with torch int64 ops, so
  ``w_rows(..., device="cuda")`` and ``w_rows(..., device="cpu")`` are bit-identical: the GPU fills its
  (possibly 20 GB) shard in place, the oracle regenerates just the rows it needs.
  Value: ((u >> 8) + 0.5) * 2^-23 - 1, exactly representable in fp32, uniform in (-1, 1).
* x and labels are small and made on the host with numpy's seeded generator, then copied.
"""
import numpy as np
import torch

_M32 = 0xFFFFFFFF
_MUL = 0x45D9F3B  # < 2^31 so that (x < 2^32) * _MUL < 2^63 never overflows int64


def _mix(x):
    x = x ^ (x >> 16)
    x = (x * _MUL) & _M32
    x = x ^ (x >> 16)
    x = (x * _MUL) & _M32
    return x ^ (x >> 16)


def _u32(seed, tag, rows, cols):
    """uint32 hash (held in int64) of (seed, tag, row, col). rows: (R,1) int64, cols: (1,D) int64."""
    h = _mix(torch.full_like(rows, (int(seed) & _M32) ^ ((int(tag) * 0x9E3779B1) & _M32)))
    h = _mix((h + (rows & _M32)) & _M32)
    h = _mix((h + (rows >> 32)) & _M32)
    return _mix((h + cols) & _M32)


def w_rows(seed, ids, d, device="cpu", tag=1):
    """Rows `ids` (global class ids) of the synthetic W (row j = class centre j), float32 (len x d)."""
    ids = torch.as_tensor(ids, dtype=torch.int64, device=device).reshape(-1, 1)
    cols = torch.arange(d, dtype=torch.int64, device=device).reshape(1, -1)
    u = _u32(seed, tag, ids, cols)
    num = 2 * (u >> 8) + 1 - (1 << 24)            # odd, |num| < 2^24: exact in fp32
    return num.to(torch.float32) * (2.0 ** -24)


def fill_w_shard(out, seed, start, tag=1, chunk=1 << 16):
    """Fill a (C_local x d) float32 tensor (any device) with rows [start, start + C_local) of W."""
    n, d = out.shape
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        ids = torch.arange(start + r0, start + r1, dtype=torch.int64, device=out.device)
        out[r0:r1] = w_rows(seed, ids, d, device=out.device, tag=tag)
    return out


def w_rows_np(seed, ids, d, tag=1):
    """Same rows as float64 numpy (exact copies of the float32 values)."""
    return w_rows(seed, np.asarray(ids, dtype=np.int64), d, tag=tag).numpy().astype(np.float64)


def make_labels(seed, step, world, B, C, mode="uniform", stress_range=None):
    """Global-batch labels (world x B). 'uniform': iid over [0, C) (P:322 Glint360K-like uniform ids).
    'stress': every label in [0, stress_range) (all in shard 0) to force k_i = |P_i|."""
    g = np.random.default_rng([int(seed), int(step), 7])
    if mode == "uniform":
        y = g.integers(0, C, size=(world, B), dtype=np.int64)
    elif mode == "stress":
        y = g.integers(0, int(stress_range), size=(world, B), dtype=np.int64)
    elif mode == "distinct":
        y = g.choice(C, size=world * B, replace=False).astype(np.int64).reshape(world, B)
    else:
        raise ValueError(mode)
    return [y[i].copy() for i in range(world)]


def make_features(seed, step, world, B, d, labels=None, dist="init", sigma=0.045, w_seed=None):
    """Per-rank features x_i (world x B x d float32).
    'init'   : iid standard normal directions (cos ~ N(0, 1/d)), norms ~ sqrt(d).
    'trained': x_n = w_{y_n}/||w_{y_n}|| + sigma * eps (CA_pcc regime of Fig.3); needs labels."""
    g = np.random.default_rng([int(seed), int(step), 11])
    eps = g.standard_normal((world, B, d))
    if dist == "init":
        x = eps
    elif dist == "trained":
        y = np.concatenate(labels)
        w = w_rows_np(w_seed if w_seed is not None else seed, y, d)
        w = w / np.linalg.norm(w, axis=1, keepdims=True)
        x = w.reshape(world, B, d) + sigma * eps
    else:
        raise ValueError(dist)
    x = x.astype(np.float32)
    return [x[i].copy() for i in range(world)]
