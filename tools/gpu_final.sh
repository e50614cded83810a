#!/bin/bash
# Round-end evidence (round 2): GPU tests with the parity log, smoke, the
# default bench line (C4 headline + C1 secondary with CPU baselines), the
# driver-style K=20 line, the reference arm, the other workloads, the ncu
# launch list of the bench command and one `ncu --set full` capture of the
# hot kernels at C4.
O=gpurun_out/final
mkdir -p $O
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=30 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_k20.json 2> $O/bench_k20.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
for w in c0 c1 c2 c3; do
  timeout 900 python bench.py --workload $w --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 900 $CMD > $O/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"estep|colsum|rowdot|zreduce|transform_sigma|sigma_final|list|bbox|init_state|mstep_fused|spectral_rank|gram|topk|gaussian|transpose" -c 300 --csv \
   --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu exit $?" >> $O/ncu_launch.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"estep_col_kernel|estep_row_kernel|rowdot_bulk|colsum_bulk|estep_col_combine|estep_row_combine" -s 40 -c 6 -o $O/hot_c4 $CMD > $O/ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/ncu_full.log
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED" $O/pytest_gpu.txt | head; tail -1 $O/smoke.txt
for f in $O/bench_*.json; do echo "== $f"; cut -c1-300 $f; done
tail -1 $O/ncu_launch.log; tail -2 $O/ncu_full.log
