#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
FCPD_COLSUM=ldg timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-calls 0 > gpurun_out/bench_ldg.json 2>> gpurun_out/bench.err
tail -4 gpurun_out/pytest_gpu.txt; python -c "
import json
for f in ['gpurun_out/bench.json','gpurun_out/bench_ldg.json']:
    try:
        d=json.load(open(f)); print(f, round(d['value'],1), d['phase_ms'], round(d['roofline']['frac'],3), d['e2e']['value'])
    except Exception as e: print(f, 'ERR', e)
"; tail -3 gpurun_out/bench.err
