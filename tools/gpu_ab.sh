#!/bin/bash
# GPU tests + bench lines of the given workloads (A/B of an E-step change).
mkdir -p gpurun_out/ab
O=gpurun_out/ab
rm -f $O/parity.jsonl
if [ "${TESTS:-1}" = 1 ]; then
  FCPD_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.txt
  tail -3 $O/pytest_gpu.txt; grep -E "^FAILED|^E " $O/pytest_gpu.txt | head -8 | cut -c1-250
fi
for w in ${WORKLOADS:-c1 c2 c4}; do
  timeout 900 python bench.py --workload $w --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
  python -c "
import json
d=json.load(open('$O/bench_$w.json'))
print('$w', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'frac %.3f' % d['roofline']['frac'], 'eval', [round(v,3) for v in d['roofline']['evaluated_frac']], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -5 $O/bench_$w.err
done
