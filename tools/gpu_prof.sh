#!/bin/bash
# tests + bench + launch list + one ncu --set full capture of the hot kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
   -k regex:"estep|colsum|zreduce|transform_sigma|sigma_final" -c 60 --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k regex:"estep_col_kernel|estep_row_kernel|colsum_kernel" -s 8 -c 4 \
   -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
tail -12 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -3 gpurun_out/ncu_full.log
