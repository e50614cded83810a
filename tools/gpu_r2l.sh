#!/bin/bash
# Round-2 pass L: row-sharded top-K products in rank groups (loopback).
O=gpurun_out/r2l
mkdir -p $O
export FCPD_TOPK_LOG=1
timeout 1500 python -m pytest tests/test_loopback.py -q -m gpu -s -rA > $O/pytest_loopback.txt 2>&1
echo "pytest exit $?" >> $O/pytest_loopback.txt
tail -3 $O/pytest_loopback.txt; grep -E "^FAILED|Error|world|topk:" $O/pytest_loopback.txt | head -40
