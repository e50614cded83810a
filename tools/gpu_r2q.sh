#!/bin/bash
# Round-2 pass Q: C0 launch list (per-kernel times) and a C0 bench line.
O=gpurun_out/r2q
mkdir -p $O
timeout 600 python bench.py --workload c0 --secondary none --steps 50 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"estep|mstep|list|bbox|init_state|rowdot|colsum|transform|sigma|zreduce|spectral" -c 120 --csv --log-file $O/launches_c0.csv python bench.py --workload c0 --secondary none --steps 5 --warmup 3 --no-cpu --e2e-calls 0 > $O/ncu_c0.log 2>&1
python -c "
import json
d=json.loads(open('$O/bench_c0.json').read().strip().splitlines()[-1])
print(d['value'], d['phase_ms'], d.get('gpu_launches'), d.get('e2e',{}).get('value'))
"
tail -2 $O/ncu_c0.log
