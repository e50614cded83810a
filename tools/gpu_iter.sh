#!/bin/bash
# iteration GPU session: tests, bench, e2e probe
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; cat gpurun_out/e2e_probe.txt
