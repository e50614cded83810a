#!/bin/bash
# Round-2 pass O: blocked Qᵀ layout (one 32 KB copy per stream unit) —
# M-step parity, C3/C4 stream times, ncu of the two stream kernels at C4.
O=gpurun_out/r2o
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_parity_full.py tests/test_loopback.py -q -m gpu -k "mstep or c3 or c4 or lowrank or loopback or streaming" -rA > $O/pytest.txt 2>&1
echo "pytest exit $?" >> $O/pytest.txt
for w in c4 c3; do
  timeout 900 python bench.py --workload $w --secondary none --steps 100 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rowdot_bulk|colsum_bulk" -s 10 -c 2 -o $O/streams_c4 python bench.py --workload c4 --secondary none --steps 3 --warmup 3 --no-cpu --e2e-calls 1 > $O/ncu.log 2>&1
tail -3 $O/pytest.txt; grep -E "^FAILED|Error" $O/pytest.txt | head
for f in $O/bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['value'], d['phase_ms'], d['roofline_hbm']['this_run'])
"; done
tail -2 $O/ncu.log
