#!/bin/bash
# first GPU session: environment, pipe microbench, GPU tests, bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/env.txt 2>&1
nproc >> gpurun_out/env.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/env.txt; free -g >> gpurun_out/env.txt
timeout 120 ./tools/pipes > gpurun_out/pipes.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err; cat gpurun_out/pipes.txt
