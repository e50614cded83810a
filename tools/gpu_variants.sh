#!/bin/bash
# A/B of library variants / env knobs:  VARIANTS="name:ENV=..:lib ..." WORKLOADS="c4 c1"
O=gpurun_out/var
mkdir -p $O
for w in ${WORKLOADS:-c4 c1}; do
for v in ${VARIANTS}; do
  name=${v%%:*}; rest=${v#*:}; envs=${rest%%:*}; libv=${rest#*:}
  L=""; [ -n "$libv" ] && L="FCPD_LIB=$PWD/paper_2006_06281_b200/variants/$libv/libfcpd_b200.so"
  env $envs $L timeout 600 python bench.py --workload $w --warmup 5 --no-cpu --e2e-calls 0 --secondary none ${BENCH_ARGS} > $O/bench_${w}_$name.json 2> $O/bench_${w}_$name.err
  python -c "
import json
d=json.load(open('$O/bench_${w}_$name.json'))
print('$w $name', 'it/s %.1f' % d['value'], 'frac %.3f' % d['roofline']['frac'], {k: round(v,4) for k,v in d['phase_ms'].items()})
" || tail -3 $O/bench_${w}_$name.err
done; done
