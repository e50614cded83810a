#!/bin/bash
# ncu launch list (per-kernel durations) of the E-step/M-step kernels of a
# short bench run, after the same command exits 0 without ncu.  NAME, CMD.
mkdir -p gpurun_out
NAME=${NAME:-launches}
CMD=${CMD:-python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0}
timeout 600 $CMD > gpurun_out/$NAME.plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/$NAME.plain.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k regex:"${KREGEX:-estep|colsum|zreduce|transform_sigma|sigma_final|list|bbox|bminmax}" -c ${COUNT:-80} --csv \
   --log-file gpurun_out/$NAME.csv $CMD > gpurun_out/$NAME.ncu.log 2>&1
echo "ncu exit $?"
