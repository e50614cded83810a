#!/bin/bash
# GPU tests (default: spectral truncation on) + A/B benches with it off.
mkdir -p gpurun_out/trunc
O=gpurun_out/trunc
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.txt 2>&1
echo "gpu tests exit $?"; tail -2 $O/pytest_gpu.txt; grep -E "^FAILED|^E " $O/pytest_gpu.txt | head -8 | cut -c1-250
cut -c1-170 $O/parity.jsonl
for tau in default 0; do
  for w in ${WORKLOADS:-c0 c1 c3}; do
    if [ $tau = default ]; then unset FCPD_SPECTRAL_TAU; else export FCPD_SPECTRAL_TAU=$tau; fi
    timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_${w}_tau$tau.json 2> $O/bench_${w}_tau$tau.err
    python -c "
import json
d=json.load(open('$O/bench_${w}_tau$tau.json'))
print('$w tau=$tau', 'it/s %.1f' % d['value'], 'e2e %.1f' % d['e2e']['value'], 'keff', d.get('spectral_rank_last'), 'hbm frac %.2f' % d['roofline']['frac'], 'sigma2 %.9g' % d['sigma2_last'], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -5 $O/bench_${w}_tau$tau.err
  done
done
