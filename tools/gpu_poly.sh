#!/bin/bash
# A/B of FCPD_EX2_POLY (pass-1 ex2 on the FMA pipe for POLY of 8 staged points)
O=gpurun_out/poly
mkdir -p $O
for w in c4 c1; do
for p in 0 1 2 3; do
  FCPD_EX2_POLY=$p timeout 600 python bench.py --workload $w --warmup 5 --no-cpu --e2e-calls 0 --secondary none > $O/bench_${w}_$p.json 2> $O/bench_${w}_$p.err
  python -c "
import json
d=json.load(open('$O/bench_${w}_$p.json'))
print('$w poly $p', 'it/s %.1f' % d['value'], 'frac %.3f' % d['roofline']['frac'], {k: round(v,4) for k,v in d['phase_ms'].items() if k.startswith('estep')})
" || tail -3 $O/bench_${w}_$p.err
done; done
