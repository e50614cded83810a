#!/bin/bash
# ncu launch list (gpu__time_duration) of the EM-iteration kernels at C4 and C0
O=gpurun_out/ll
mkdir -p $O
for w in c4 c0; do
  CMD="python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
  timeout 900 $CMD > $O/plain_$w.log 2>&1 || { echo "plain $w failed"; tail -3 $O/plain_$w.log; continue; }
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"estep|colsum|rowdot|zreduce|transform_sigma|sigma_final|list|bbox|mstep_fused|small_iter|spectral_rank" -c 300 --csv --log-file $O/launches_$w.csv $CMD > $O/ncu_$w.log 2>&1
  echo "ncu $w exit $?"
  python tools/launch_means.py $O/launches_$w.csv | head -16
done
