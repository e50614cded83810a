#!/bin/bash
# GPU tests (centred form, parity log) + A/B of the E-step pair forms.
mkdir -p gpurun_out/form
O=gpurun_out/form
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1
tail -2 $O/pytest_gpu.txt; grep -E "^FAILED|^E " $O/pytest_gpu.txt | head -8 | cut -c1-300
cut -c1-200 $O/parity.jsonl
for form in ${FORMS:-centred diff}; do
  for w in ${WORKLOADS:-c1 c2 c4}; do
    FCPD_ESTEP_FORM=$form timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_${w}_$form.json 2> $O/bench_${w}_$form.err
    python -c "
import json
d=json.load(open('$O/bench_${w}_$form.json'))
r=d['estep_roofline']
print('$w $form', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'estep frac %.3f' % r['frac'], 'eval', [round(x,3) for x in r['evaluated_frac']], 'sigma2 %.6g' % d['sigma2_last'], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -5 $O/bench_${w}_$form.err
  done
done
