#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl
FCPD_PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu -rA > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
grep -E "passed|failed" gpurun_out/pytest_gpu.txt | tail -3; grep -E "^FAILED|var rel" gpurun_out/pytest_gpu.txt | head -20; cat gpurun_out/parity.jsonl
