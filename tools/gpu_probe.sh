#!/bin/bash
# Culling-bound A/B: parity of the culled path, per-iteration traces with the
# probe bound on/off, and the bench lines of every workload.
O=gpurun_out/probe
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -s -k "culling or estep or full_size" > $O/pytest.txt 2>&1
echo "pytest exit $?" >> $O/pytest.txt
for w in ${WORKLOADS:-c1 c2 c4}; do
  for pr in 1 0; do
    FCPD_CULL_PROBE=$pr timeout 600 python tools/cull_trace.py $w > $O/trace_${w}_p$pr.json 2> $O/trace_${w}_p$pr.err
  done
done
tail -3 $O/pytest.txt
grep -h "σ² rel\|late tile" $O/pytest.txt
for f in $O/trace_*.json; do python -c "import json,sys; d=json.load(open('$f')); t=d['trace']; print('$f', round(d['it_per_s'],1), [round(r['f1'],3) for r in t[::10]], [round(r['f2'],3) for r in t[::10]])"; done
