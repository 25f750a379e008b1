#!/bin/bash
# one gpurun call: GPU test suite (measured parity errors logged), then the default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
PFC_PARITY_LOG=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -5 gpurun_out/pytest.log
