#!/bin/bash
# C1 per-kernel launch times (ncu, serialised) + the fused M-step phase probe
O=gpurun_out/c1
mkdir -p $O
CMD="python bench.py --workload c1 --steps 8 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err || { tail $O/plain.err; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"estep|mstep|list|bbox|combine" -c 200 --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1
echo "ncu exit $?"
python tools/launch_means.py $O/launches.csv 2>/dev/null | head -20
FCPD_LIB=$PWD/paper_2006_06281_b200/variants/probe/libfcpd_b200.so timeout 300 $CMD 2>&1 | grep probe | head -3
