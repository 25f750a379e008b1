"""Partial FC oracle: plain, slow, float64 CPU implementation of the paper's method.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module. The product path (paper_2010_05222_b200/) never does, and this
module shares no code, header, table or constant with it.

It follows, in the paper's order and notation:
  * Alg.1 "The Model Parallel on the i-th GPU": X = allgather(x_i); logits_i = X w_i;
    den_i = sum e^{logits_i}; den = allreduce(den_i); prob_i = e^{logits_i}/den; grad logits_i =
    prob_i - onehot_i; grad w_i = X^T grad logits_i; grad X = allreduce(grad logits_i w_i^T);
    grad x_i = get_submatrix(i, grad X).
  * Eq.5 softmax loss with bias 0, Eq.6 normalised cosine logits f_j = s cos(theta_j)
    (PAPER.md:164-169), margins CosFace m=0.4 / ArcFace m=0.5, s=64.
  * PPRN distributed sampling: 1) positives on this GPU, 2) per-GPU count,
    3) random negatives from w_i - w_i^p; W^s = [W^p, W^n] (Eq.10), sampled softmax Eq.9.
  * Momentum SGD, lazy on the sampled rows.
Every place where the paper is silent or ambiguous takes the DESIGN.md reading named in the comment
(R1..R20, mirroring SURVEY.md §8(c)).

All ranks i = 0..k-1 are simulated in one process; collectives are rank-ordered concatenation and
rank-ascending sums (the single-matrix form of Alg.1).

Pinned in tests/test_oracle_pins.py (closed forms, library special cases, finite differences,
identities, brute force). Parity beyond those pins is "parity unpinned" only for bf16-scale values,
which the paper does not print (see DESIGN.md §Oracle pins).
"""
import math
from dataclasses import dataclass

import numpy as np

from .philox import class_key

MARGIN_NONE, MARGIN_ARCFACE, MARGIN_COSFACE = 0, 1, 2
# Sampling rules (R1, R23, R24):
#   SAMPLE_PPRN        north_star: k_i = max(ceil(r C_local), |P_i|), positives always kept
#   SAMPLE_PPRN_PAPER  the paper's literal step 2: s_i = (|w_i| - |w_i^p|) r negatives, rounded
#                      half up; k_i = |P_i| + s_i
#   SAMPLE_RANDOM      fully random (the Fig.3 baseline): ceil(r C_local) classes drawn from the
#                      whole shard ignoring the labels; positives may be missing
SAMPLE_PPRN, SAMPLE_PPRN_PAPER, SAMPLE_RANDOM = 0, 1, 2
NORM_EPS = 1e-12          # R8: divide by max(||v||, 1e-12)
ARC_DERIV_EPS = 1e-6      # R10: guard of the ArcFace derivative at cos -> +-1


@dataclass
class OracleConfig:
    num_classes: int          # C
    dim: int                  # d
    batch: int                # N = B, per rank (equal on every rank)
    world_size: int = 1       # k
    sample_rate: float = 1.0  # r
    scale: float = 64.0       # s
    margin_type: int = MARGIN_ARCFACE
    margin: float = 0.5       # ArcFace 0.5 / CosFace 0.4
    momentum: float = 0.9     # mu (R15)
    weight_decay: float = 0.0 # lambda (R15, explicit)
    seed: int = 0
    sample_mode: int = SAMPLE_PPRN
    ignore_index: bool = False  # R28: a label of -1 marks an ignored row (PyTorch ignore_index = -1)


# ----------------------------------------------------------------------------------------------
# Partition and sampling
# ----------------------------------------------------------------------------------------------
def shard_range(C, k, i):
    """W is "evenly divided into different GPUs according to the order".
    R6: balanced, the first C mod k ranks get one extra class. Returns (a_i, C_local(i))."""
    base, extra = divmod(C, k)
    a = i * base + min(i, extra)
    return a, base + (1 if i < extra else 0)


def sample_budget(r, C_local):
    """R1 (north_star): per-shard sampled count target ceil(r * C_local), computed as the IEEE double
    expression ceil((double) r * (double) C_local). |S| = C*r (Eq.9), equal per GPU
    (PAPER.md:293)."""
    return int(math.ceil(float(r) * float(C_local)))


def positives(Y, a, C_local):
    """Step 1: positive class centres on this GPU = labels in [a, a + C_local),
    deduplicated (R5), ascending."""
    Y = np.asarray(Y, dtype=np.int64)
    return np.unique(Y[(Y >= a) & (Y < a + C_local)])


def paper_budget(r, C_local, npos):
    """The paper's step 2: s_i = (|w_i| - |w_i^p|) * r negatives; the product is rounded half up
    (floor(x + 0.5) of the IEEE double product) and clamped to [0, |w_i| - |w_i^p|] (R23)."""
    n = int(math.floor(float(C_local - npos) * float(r) + 0.5))
    return min(max(n, 0), C_local - npos)


def sample_shard(Y, a, C_local, r, seed, step, mode=SAMPLE_PPRN):
    """Steps 1-3 of the distributed approximation on one shard.

    k_i = max(ceil(r C_local), |P_i|) (R1); n_i = k_i - |P_i| negatives are "randomly sampled" from
    w_i - w_i^p (step 3). R2/R3: the n_i negatives with the smallest (h_j, j), h_j = Philox key of the
    global class id j. R4: the sampled set is returned in ascending global id order.
    mode SAMPLE_PPRN_PAPER: n_i = paper_budget (R23). mode SAMPLE_RANDOM: no positives are kept; the
    ceil(r C_local) classes with the smallest (h_j, j) over the whole shard (R24).
    Returns (idx int64 ascending global ids, number of positives kept)."""
    P = positives(Y, a, C_local)
    if mode == SAMPLE_RANDOM:
        P = P[:0]
        k_i = sample_budget(r, C_local)
    elif mode == SAMPLE_PPRN_PAPER:
        k_i = len(P) + paper_budget(r, C_local, len(P))
    else:
        k_i = max(sample_budget(r, C_local), len(P))
    n_i = k_i - len(P)
    U = np.setdiff1d(np.arange(a, a + C_local, dtype=np.int64), P)     # w_i - w_i^p
    h = class_key(U, seed, step)
    order = np.lexsort((U, h))                                          # primary h, ties: smaller j
    N = U[order[:n_i]]
    return np.sort(np.concatenate([P, N])), len(P)


# ----------------------------------------------------------------------------------------------
# Normalisation and margins (Eq.6; margins PAPER.md:330)
# ----------------------------------------------------------------------------------------------
def normalize_rows(v):
    """l2-normalise rows. R8: divide by max(||v||, 1e-12). Returns (v_hat, ||v||)."""
    v = np.asarray(v, dtype=np.float64)
    n = np.sqrt(np.sum(v * v, axis=1))
    return v / np.maximum(n, NORM_EPS)[:, None], n


def margin_phi(c, margin_type, m):
    """Target-logit margin before scaling. ArcFace: cos(theta + m) with theta = arccos(c); R9: when
    theta + m >= pi (c <= cos(pi - m)) use c - m sin m. CosFace: c - m. None: c."""
    c = np.asarray(c, dtype=np.float64)
    if margin_type == MARGIN_NONE:
        return c.copy()
    if margin_type == MARGIN_COSFACE:
        return c - m
    cc = np.clip(c, -1.0, 1.0)
    theta = np.arccos(cc)
    return np.where(theta + m < math.pi, np.cos(theta + m), c - m * math.sin(m))


def margin_dphi(c, margin_type, m):
    """d phi / d c. ArcFace main branch: d/dc cos(arccos c + m) = sin(theta + m) / sin(theta), with
    sin(theta) = sqrt(1 - c^2) guarded below by 1e-6 (R10); fallback branch: 1. CosFace / none: 1."""
    c = np.asarray(c, dtype=np.float64)
    if margin_type != MARGIN_ARCFACE:
        return np.ones_like(c)
    cc = np.clip(c, -1.0, 1.0)
    theta = np.arccos(cc)
    sin_theta = np.maximum(np.sqrt(np.maximum(0.0, 1.0 - cc * cc)), ARC_DERIV_EPS)
    return np.where(theta + m < math.pi, np.sin(theta + m) / sin_theta, 1.0)


# ----------------------------------------------------------------------------------------------
# Forward + backward of the sampled, model-parallel layer (Alg.1 with PPRN)
# ----------------------------------------------------------------------------------------------
def forward_backward(cfg, xs, ys, w_rows, step=0, keep_intermediates=False):
    """One Alg.1 pass over all k simulated ranks with PPRN sampling.

    xs: list of k arrays (B x d) — x_i, features on GPU i.  ys: list of k int arrays (B) — labels.
    w_rows(global_ids) -> (len x d) array: rows of W (row j = class centre j, D1).
    step: the iteration counter that keys the sampler (R2).
    Returns a dict with loss, grad_x (list per rank), idx (list per rank), k (list), dW (list per rank,
    k_i x d, gradient w.r.t. the raw W rows), lse (M), target_cos (M).
    """
    k, B, d, C = cfg.world_size, cfg.batch, cfg.dim, cfg.num_classes
    s, mt, m = float(cfg.scale), cfg.margin_type, float(cfg.margin)
    assert len(xs) == k and len(ys) == k
    # Alg.1 L2: X = allgather(x_i) — rank-ordered concatenation; labels likewise (P:297 needs them).
    X = np.concatenate([np.asarray(x, dtype=np.float64).reshape(B, d) for x in xs], axis=0)
    Y = np.concatenate([np.asarray(y, dtype=np.int64).reshape(B) for y in ys], axis=0)
    M = k * B
    # R28: with ignore_index, rows labelled -1 take no part in Eq.5 — no loss term, no
    # gradient, no positive class — and the mean runs over the M_valid other rows
    ign = (Y == -1) if cfg.ignore_index else np.zeros(M, dtype=bool)
    if np.any(((Y < 0) | (Y >= C)) & ~ign):
        raise ValueError("label outside [0, C) (R7)")
    M_valid = max(int(np.sum(~ign)), 1)
    Xh, xnorm = normalize_rows(X)                                    # Eq.6: fix ||x|| by l2 normalisation

    # PPRN steps 1-3 on every shard, then W^s = [w_1^s, ..., w_k^s] (Eq.10) in rank order.
    idx, kk, npos = [], [], []
    for i in range(k):
        a, Cl = shard_range(C, k, i)
        ii, npi = sample_shard(Y, a, Cl, cfg.sample_rate, cfg.seed, step, cfg.sample_mode)
        idx.append(ii); kk.append(len(ii)); npos.append(npi)
    S = np.concatenate(idx)                                          # global ids of the sampled set
    Wraw = np.asarray(w_rows(S), dtype=np.float64).reshape(len(S), d)
    Wh, wnorm = normalize_rows(Wraw)                                 # Eq.6: fix ||w_j|| by l2 normalisation

    # Alg.1 L3 (sampled): cosines, then the margin at each row's positive column (R11).
    cos = Xh @ Wh.T                                                  # M x |S|
    col_of = {int(g): t for t, g in enumerate(S)}
    tcol = np.array([col_of.get(int(y), -1) for y in Y], dtype=np.int64)   # -1: positive not sampled (R24)
    rows = np.arange(M)
    hit = tcol >= 0
    # cos(theta) between each row and its own class centre (sampled or not): Eq.7's CA_pcc and z_t
    Wy, _ = normalize_rows(np.asarray(w_rows(np.where(ign, 0, Y)), dtype=np.float64).reshape(M, d))
    ct = np.where(ign, 0.0, np.sum(Xh * Wy, axis=1))
    zt = s * margin_phi(ct, mt, m)
    Z = s * cos
    Z[rows[hit], tcol[hit]] = zt[hit]

    # Alg.1 L5-8: den_i, den = allreduce(den_i), prob = e^logits / den; R12: shift by the global row max.
    zmax = np.max(Z, axis=1)
    den = np.sum(np.exp(Z - zmax[:, None]), axis=1)
    lse = zmax + np.log(den)
    prob = np.exp(Z - lse[:, None])
    # Eq.5 (R13: mean over the global batch M = N k). A row whose positive is not in S (fully random, R24)
    # keeps Eq.9's denominator over S and its own positive logit as numerator.
    # R28: ignored rows are left out of the mean (M_valid = M without ignore_index)
    loss = float(np.sum(np.where(ign, 0.0, lse - zt)) / M_valid)
    ca_pcc = float(np.sum(ct) / M_valid)                             # Eq.7 (ct = 0 on ignored rows)

    # Alg.1 L9: grad logits = prob - onehot, times dL/dlogits scale 1/M, chained through
    # z = s * phi(c) at the target and z = s * c elsewhere. R24: no onehot term (no positive pull) when the
    # positive is not sampled.
    onehot = np.zeros_like(prob)
    onehot[rows[hit], tcol[hit]] = 1.0
    G = (prob - onehot) / M_valid                                    # dL/dZ
    G[ign] = 0.0                                                     # R28: an ignored row has no gradient
    Gc = s * G                                                       # dL/dcos, non-target columns
    Gc[rows[hit], tcol[hit]] *= margin_dphi(ct[hit], mt, m)

    # Alg.1 L10: grad w = X^T grad logits ; L12: grad X = allreduce(grad logits w^T) (sum over ranks is
    # the sum over the concatenated sampled columns); R14: analytic backprop through both l2 norms.
    dXh = Gc @ Wh                                                    # M x d
    dWh = Gc.T @ Xh                                                  # |S| x d
    gx = (dXh - Xh * np.sum(Xh * dXh, axis=1, keepdims=True)) / np.maximum(xnorm, NORM_EPS)[:, None]
    gw = (dWh - Wh * np.sum(Wh * dWh, axis=1, keepdims=True)) / np.maximum(wnorm, NORM_EPS)[:, None]

    out = {
        "loss": loss, "ca_pcc": ca_pcc,
        "grad_x": [gx[i * B:(i + 1) * B] for i in range(k)],         # Alg.1 L13: get_submatrix(i, grad X)
        "idx": idx, "k": kk, "num_pos": npos,
        "dW": [], "lse": lse, "target_cos": ct, "tcol": tcol,
    }
    off = 0
    for i in range(k):
        out["dW"].append(gw[off:off + kk[i]])
        off += kk[i]
    if keep_intermediates:
        out.update(cos=cos, Z=Z, prob=prob, Gc=Gc, S=S, Wh=Wh, Xh=Xh)
    return out


def sgd_momentum_rows(W_rows, V_rows, dW, lr, momentum, weight_decay):
    """Momentum SGD (W, its gradient and the momentum buffer = 12 bytes per parameter),
    PyTorch form without dampening or Nesterov (R15): v <- mu v + g + lambda w ; w <- w - lr v.
    Applied lazily to the sampled rows only; untouched rows keep W and V unchanged (R15).
    Returns the updated (W_rows, V_rows)."""
    W_rows = np.asarray(W_rows, dtype=np.float64)
    V_rows = np.asarray(V_rows, dtype=np.float64)
    V_new = momentum * V_rows + np.asarray(dW, dtype=np.float64) + weight_decay * W_rows
    return W_rows - lr * V_new, V_new


# ----------------------------------------------------------------------------------------------
# Row / column spot checks for sizes where the full M x |S| matrices are too large to keep
# ----------------------------------------------------------------------------------------------
def spot_rows(cfg, X, Y, S, w_rows, rows, step_unused=None):
    """For the chosen batch rows n: (lse_n, loss term lse_n - z_{n,y_n}, grad_x_n) of the same
    definitions as forward_backward, computed one row at a time over the full sampled set S (the
    union of all ranks' idx). X: (M x d) all features, Y: (M) labels, S: ascending-per-rank sampled ids.
    Used by full-size parity tests; identical arithmetic to forward_backward restricted to a row."""
    s, mt, m = float(cfg.scale), cfg.margin_type, float(cfg.margin)
    M = X.shape[0]
    Wh, _ = normalize_rows(w_rows(S))
    res = []
    for n in rows:
        xh, xn = normalize_rows(X[n:n + 1])
        c = (Wh @ xh[0])                                             # |S|
        t = int(np.nonzero(S == Y[n])[0][0])
        z = s * c
        z[t] = s * margin_phi(c[t:t + 1], mt, m)[0]
        zmax = z.max()
        lse = zmax + math.log(np.sum(np.exp(z - zmax)))
        p = np.exp(z - lse)
        gc = s * p / M
        gc[t] = s * (p[t] - 1.0) / M * margin_dphi(c[t:t + 1], mt, m)[0]
        dxh = gc @ Wh
        gx = (dxh - xh[0] * np.dot(xh[0], dxh)) / max(xn[0], NORM_EPS)
        res.append((lse, lse - z[t], gx))
    return res


def row_lse(cfg, Xh, Y, S, Wh, block=64):
    """lse_n = log sum_{j in S} e^{z_nj} (R12: shifted by the row max) and the target cosine c_t for every row n,
    with z = s c except z_t = s phi(c_t) (R11) — the same definitions as forward_backward, evaluated for `block`
    rows at a time so that the M x |S| cosine matrix never has to exist at once (C5: 2048 x 1.25M). Each row's
    sum still runs over the whole of S in one np.sum."""
    s, mt, m = float(cfg.scale), cfg.margin_type, float(cfg.margin)
    pos = {int(g): t for t, g in enumerate(S)}
    tcol = np.array([pos[int(y)] for y in Y])
    M = Xh.shape[0]
    lse, ct = np.empty(M), np.empty(M)
    for r0 in range(0, M, block):
        r1 = min(M, r0 + block)
        rows = np.arange(r1 - r0)
        z = s * (Xh[r0:r1] @ Wh.T)                                   # block x |S|
        ct[r0:r1] = z[rows, tcol[r0:r1]] / s
        z[rows, tcol[r0:r1]] = s * margin_phi(ct[r0:r1], mt, m)
        zmax = z.max(axis=1)
        lse[r0:r1] = zmax + np.log(np.sum(np.exp(z - zmax[:, None]), axis=1))
    return lse, ct, tcol


def spot_cols(cfg, X, Y, S, w_rows, cols):
    """Gradient w.r.t. the raw W rows of the sampled classes S[cols] (same definitions as forward_backward:
    Alg.1 L10 grad w = X^T grad logits, then the l2-norm backprop R14), for sizes where only a few columns are
    wanted. The row log-sum-exps need every row over the whole sampled set S (row_lse).
    Returns (dW rows for cols, lse for every row, target cosine for every row)."""
    s, mt, m = float(cfg.scale), cfg.margin_type, float(cfg.margin)
    M = X.shape[0]
    Xh, _ = normalize_rows(X)
    Wraw = np.asarray(w_rows(S), dtype=np.float64)
    Wh, _ = normalize_rows(Wraw)
    lse, ct, tcol = row_lse(cfg, Xh, Y, S, Wh)
    out = []
    for t in cols:
        c = Xh @ Wh[t]                                               # cosines of every row with class S[t]
        hit = tcol == t
        c[hit] = margin_phi(ct[hit], mt, m)                          # z / s (margin at the target, R11)
        gc = s * np.exp(s * c - lse) / M                             # dL/dcos for non-target rows
        gc[hit] = s * (np.exp(s * c[hit] - lse[hit]) - 1.0) / M * margin_dphi(ct[hit], mt, m)
        dwh = gc @ Xh
        wr = Wraw[t]
        wn = np.sqrt(np.sum(wr * wr))
        wh = wr / max(wn, NORM_EPS)
        out.append((dwh - wh * np.dot(wh, dwh)) / max(wn, NORM_EPS))
    return np.array(out), lse, ct
