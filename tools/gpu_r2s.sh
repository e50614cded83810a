#!/bin/bash
# Round-2 pass S: combine kernels with several threads per point — parity,
# C1/C4 benches, ncu of the combines at C1.
O=gpurun_out/r2s
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest.txt 2>&1
echo "pytest exit $?" >> $O/pytest.txt
timeout 900 python bench.py --workload c1 --secondary none --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_c1_k20.json 2> $O/bench_c1_k20.err
timeout 900 python bench.py --workload c1 --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --workload c0 --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"combine" -s 20 -c 2 -o $O/combine_c1 python bench.py --workload c1 --secondary none --steps 3 --warmup 3 --no-cpu --e2e-calls 0 > $O/ncu.log 2>&1
tail -3 $O/pytest.txt; grep -E "^FAILED" $O/pytest.txt | head
for f in $O/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value'],1), 'estep', round(r['estep_ms_per_iteration'],4), 'frac', round(r['frac'],3), d['phase_ms'])
"; done
