#!/bin/bash
timeout 1200 python -m pytest tests -q -x -m gpu > gpurun_out/t.txt 2>&1; tail -1 gpurun_out/t.txt; grep -E "^E " gpurun_out/t.txt | head -5
for rp in 2 1; do
  FCPD_ROW_PAIRS=$rp NAME=rp$rp KREGEX="estep_row_kernel" COUNT=6 bash tools/gpu_launches.sh > /dev/null 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/rp$rp.csv')) if len(r)>10]
hdr=rows[0]; vi=hdr.index('Metric Value')
v=[float(r[vi].replace(',',''))/1000 for r in rows[1:]]
print('row_pairs=$rp', ['%.1f' % x for x in v[-3:]])
PY
  for w in c1 c4; do
    FCPD_ROW_PAIRS=$rp timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > gpurun_out/b_${w}_$rp.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/b_${w}_$rp.json')); print('$w rp=$rp', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), {k: round(v,4) for k,v in d['phase_ms'].items()})"
  done
done
