#!/bin/bash
# ncu --set full (with source) of the two basis streams at C4
O=gpurun_out/ncu_streams
mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 900 $CMD > $O/plain.log 2>&1 || { echo "plain run failed"; tail $O/plain.log; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"rowdot_bulk|colsum_bulk" -s 6 -c 2 -o $O/streams_c4 $CMD > $O/ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/ncu_full.log
tail -2 $O/ncu_full.log
