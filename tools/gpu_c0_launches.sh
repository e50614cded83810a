#!/bin/bash
O=gpurun_out/c0
mkdir -p $O
CMD="python bench.py --workload c0 --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err || { tail $O/plain.err; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1
echo "ncu exit $?"
python tools/launch_means.py $O/launches.csv 2>/dev/null | head -30 || true
