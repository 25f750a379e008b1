"""Partial FC oracle — TEST INFRASTRUCTURE.

A plain float64 CPU implementation of the paper's definitions (arXiv 2010.05222, /root/reference/PAPER.md)
used only to check the CUDA path. Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import it; the product package never does.
"""
from .philox import philox4x32_10, class_key  # noqa: F401
from .pfc import (  # noqa: F401
    OracleConfig, MARGIN_NONE, MARGIN_ARCFACE, MARGIN_COSFACE, SAMPLE_PPRN, SAMPLE_PPRN_PAPER, SAMPLE_RANDOM, paper_budget,
    shard_range, sample_budget, positives, sample_shard, normalize_rows, margin_phi, margin_dphi,
    forward_backward, sgd_momentum_rows, spot_rows, spot_cols,
)
