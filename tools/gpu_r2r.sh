#!/bin/bash
# Round-2 pass R: ncu of the E-step combine kernels at C1.
O=gpurun_out/r2r
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"combine" -s 20 -c 2 -o $O/combine_c1 python bench.py --workload c1 --secondary none --steps 3 --warmup 3 --no-cpu --e2e-calls 0 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
