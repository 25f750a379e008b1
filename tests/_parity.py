"""Measured parity errors of the CUDA path against the oracle, collected by the -m gpu tests and printed in the
pytest terminal summary (and appended as JSON lines to $PFC_PARITY_LOG when set), so every bf16 / fp32 case
reports what it achieved against the north-star bars, not just pass / fail."""
import json
import os

ERRORS = []


def record(test, precision, **errs):
    row = {"test": test, "precision": precision}
    row.update({k: float(v) for k, v in errs.items()})
    ERRORS.append(row)
    path = os.environ.get("PFC_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(row) + "\n")
    return row
