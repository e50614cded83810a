#!/bin/bash
# ncu --set full of the two E-step pass kernels at C4 (dense phase launches).
O=gpurun_out/ncu_pass
mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 900 $CMD > $O/plain.log 2>&1 || { echo "plain run failed"; tail $O/plain.log; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"estep_col_kernel|estep_row_kernel" -s 4 -c 2 -o $O/pass_c4 $CMD > $O/ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/ncu_full.log
tail -2 $O/ncu_full.log
