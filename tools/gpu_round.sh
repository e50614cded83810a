#!/bin/bash
# Round-end evidence: GPU tests (parity log), the default bench line (c1 with
# the CPU baseline), the other workloads, the reference arm, and the ncu
# launch list of the default bench command (one ncu per call).
mkdir -p gpurun_out/round
O=gpurun_out/round
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for w in ${WORKLOADS:-c0 c2 c3 c4}; do
  timeout 900 python bench.py --workload $w --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"estep|colsum|zreduce|transform_sigma|sigma_final|list|bbox|bminmax|mstep_fused|spectral_rank" -c 80 --csv \
   --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu exit $?" >> $O/ncu_launch.log
tail -2 $O/pytest_gpu.txt; cat $O/smoke.txt | tail -1
for f in $O/bench_*.json; do echo "== $f"; cut -c1-400 $f; done
tail -1 $O/ncu_launch.log
