#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
for ch in 1 0; do
  if [ $ch = 1 ]; then export FCPD_OVERLAP_CHUNKS=1; else unset FCPD_OVERLAP_CHUNKS; fi
  for w in c1 c3; do
    timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu --e2e-calls 1 > gpurun_out/bench_${w}_$ch.json 2> gpurun_out/bench_${w}_$ch.err
    python -c "
import json
d=json.load(open('gpurun_out/bench_${w}_$ch.json'))
print('$w chunks1=$ch', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'ms/step %.4f' % d['ms_per_step'])
" || tail -5 gpurun_out/bench_${w}_$ch.err
  done
done
