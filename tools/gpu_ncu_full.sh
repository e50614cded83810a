#!/bin/bash
# One ncu --set full capture of the hot kernels of the default bench command
# (after the same command exits 0 without ncu).  NAME=report name.
mkdir -p gpurun_out
NAME=${NAME:-prof}
CMD=${CMD:-python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0}
KREGEX=${KREGEX:-estep_col_kernel|estep_row_kernel|colsum_bulk_kernel}
timeout 600 $CMD > gpurun_out/$NAME.plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/$NAME.plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:"$KREGEX" -s ${SKIP:-6} -c ${COUNT:-4} \
   -o gpurun_out/$NAME $CMD > gpurun_out/$NAME.ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/$NAME.ncu.log
