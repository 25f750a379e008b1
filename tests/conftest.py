import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (torchrun NCCL path)")


def pytest_terminal_summary(terminalreporter):
    import _parity
    if not _parity.ERRORS:
        return
    tr = terminalreporter
    tr.section("measured parity errors vs the float64 oracle (loss: relative; grad_x / dW / V: max|a-b|/max|b|)")
    for r in _parity.ERRORS:
        vals = "  ".join(f"{k}={v:.3e}" for k, v in r.items() if k not in ("test", "precision"))
        tr.write_line(f"{r['precision']:5s} {vals}  {r['test']}")
