"""The real multi-GPU path (one process per GPU, NCCL over NVLink): `torchrun --nproc-per-node N` of
tests/mgpu_worker.py, N = 2 and every GPU of the box. Each run checks the NCCL N-rank fused train step (eager,
graph-captured, replayed) against the loopback group on the same inputs — ids bit-exact, floats bit-exact at N = 2
(a + b is order-free), within 1e-6 / 1e-5 at larger N — and against the float64 oracle (ids bit-exact, north-star
bf16 bars). Skipped on boxes with fewer than 2 GPUs (this build's GPU runs have one)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("comm", ["nccl", "nccl_fused"])
@pytest.mark.parametrize("nproc", ["2", "all"])
@pytest.mark.parametrize("C,B", [(40_000, 64), (200_000, 256)], ids=["fused-M", "pair-M"])
def test_nccl_ranks_match_loopback_and_oracle(nproc, C, B, comm):
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip(f"needs >= 2 GPUs (found {n})")
    world = 2 if nproc == "2" else n
    if nproc == "all" and n == 2:
        pytest.skip("same as nproc=2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           str(C), str(B), comm]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [l for l in r.stdout.splitlines() if l.startswith("MGPU_REPORT ")]
    assert lines, r.stdout[-2000:]
    rep = json.loads(lines[-1].split(" ", 1)[1])
    assert rep["ok"] and rep["world"] == world
