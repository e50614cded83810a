#!/bin/bash
# Round-end evidence (round 2, session 2): GPU tests with the parity log,
# smoke, one `ncu --set full` capture of the hot kernels at C4 (+ the FP32 /
# XU instruction counters) summarised into profiles/r2_ncu_summary.json
# BEFORE the benches (bench.py reads roofline.traffic from it), the default
# bench line (C4 headline + C1 secondary with CPU baselines), the driver-style
# K=20 line, the reference arm, the other workloads, the ncu launch list.
O=gpurun_out/final2
mkdir -p $O
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=30 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
CMD="python bench.py --steps 5 --warmup 3 --no-cpu --e2e-calls 0 --secondary none"
timeout 900 $CMD > $O/plain.log 2>&1
M=sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__inst_executed_pipe_xu.sum
timeout 1500 ncu --set full --metrics $M --import-source on --clock-control none -k regex:"estep_col_kernel|estep_row_kernel|rowdot_bulk|colsum_bulk|estep_col_combine|estep_row_combine" -s 40 -c 6 -o $O/hot_c4 $CMD > $O/ncu_full.log 2>&1
echo "ncu full exit $?" >> $O/ncu_full.log
python tools/ncu_summarize.py $O/hot_c4.ncu-rep $O/r2_ncu_summary.json > $O/ncu_summary.txt 2>&1 && cp $O/r2_ncu_summary.json profiles/r2_ncu_summary.json
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_k20.json 2> $O/bench_k20.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
for w in c0 c1 c2 c3; do
  timeout 900 python bench.py --workload $w --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "ncu exit $?" >> $O/ncu_launch.log
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED" $O/pytest_gpu.txt | head; tail -1 $O/smoke.txt
cat $O/ncu_summary.txt
for f in $O/bench_*.json; do echo "== $f"; cut -c1-300 $f; done
tail -1 $O/ncu_launch.log; tail -2 $O/ncu_full.log
