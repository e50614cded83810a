#!/bin/bash
# Round-2 pass G: full GPU suite at q = 4, ex2-polynomial A/B (C1, C4),
# setup time vs power steps (C4), default bench line + launch list.
O=gpurun_out/r2g
mkdir -p $O
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=25 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
for p in 0 1 2 3; do
  for w in c1 c4; do
    FCPD_EX2_POLY=$p timeout 900 python bench.py --workload $w --secondary none --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/poly${p}_$w.json 2> $O/poly${p}_$w.err
  done
done
for q in 2 3; do
  FCPD_TOPK_ITERS=$q timeout 900 python bench.py --workload c4 --secondary none --steps 5 --warmup 3 --no-cpu --e2e-calls 1 > $O/topk${q}_c4.json 2> $O/topk${q}_c4.err
done
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED|Error" $O/pytest_gpu.txt | head -20
cat $O/smoke.txt | tail -2
for f in $O/*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d.get('roofline',{})
print(d['value'], d.get('setup_s'), r.get('frac'), r.get('estep_ms_per_iteration'), d.get('sigma2_last'), (d.get('e2e') or {}).get('value'))
" 2>&1 | tail -1; done
