#!/bin/bash
# Spatial-order change: GPU parity suite, then per-iteration traces.
O=gpurun_out/sort
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest.txt 2>&1
echo "pytest exit $?" >> $O/pytest.txt
for w in ${WORKLOADS:-c1 c2 c4}; do
  timeout 600 python tools/cull_trace.py $w > $O/trace_$w.json 2> $O/trace_$w.err
done
tail -3 $O/pytest.txt
for w in ${WORKLOADS:-c1 c2 c4}; do python -c "import json; d=json.load(open('$O/trace_$w.json')); t=d['trace']; print('$w', round(d['it_per_s'],1), [round(r['ms']*1000) for r in t[::10]], [round(r['f2'],3) for r in t[::10]])"; done
