#!/bin/bash
# Tensor-core pass 2 (FCPD_ESTEP_TC=1): parity tests, then A/B benches.
mkdir -p gpurun_out/tc
O=gpurun_out/tc
rm -f $O/parity.jsonl
export FCPD_ESTEP_TC=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "estep_matches_oracle or degenerate_rows or far_rows" > $O/pytest_estep.txt 2>&1
echo "estep tests exit $?"; tail -3 $O/pytest_estep.txt; grep -E "^E " $O/pytest_estep.txt | head -8 | cut -c1-250
[ "${QUICK:-0}" = "1" ] && exit 0
FCPD_PARITY_LOG=$O/parity.jsonl timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1
echo "gpu tests exit $?"; tail -2 $O/pytest_gpu.txt; grep -E "^FAILED|^E " $O/pytest_gpu.txt | head -8 | cut -c1-250
cut -c1-170 $O/parity.jsonl
for tc in 1 0; do
  for w in ${WORKLOADS:-c1 c3 c4}; do
    FCPD_ESTEP_TC=$tc timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_${w}_tc$tc.json 2> $O/bench_${w}_tc$tc.err
    python -c "
import json
d=json.load(open('$O/bench_${w}_tc$tc.json'))
r=d['estep_roofline']
print('$w tc=$tc', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'estep frac %.3f' % r['frac'], 'sigma2 %.7g' % d['sigma2_last'], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -5 $O/bench_${w}_tc$tc.err
  done
done
