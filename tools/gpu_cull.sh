#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/parity.jsonl
FCPD_PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt; grep -E "^FAILED|^E " gpurun_out/pytest_gpu.txt | head -5 | cut -c1-200
cat gpurun_out/parity.jsonl | cut -c1-160
for cull in ${CULLS:-1 0}; do
  for w in c1 c2 c4; do
    FCPD_CULL=$cull timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > gpurun_out/bench_${w}_cull$cull.json 2> gpurun_out/bench_${w}_cull$cull.err
    python -c "
import json
d=json.load(open('gpurun_out/bench_${w}_cull$cull.json'))
print('$w cull=$cull', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'ms/step %.4f' % d['ms_per_step'], 'sigma2 %.3g' % d['sigma2_last'], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -5 gpurun_out/bench_${w}_cull$cull.err
  done
done
