#!/bin/bash
# Round-2 pass D: combine kernels (with folded b ranges + fallbacks), the
# rank-group data plane (loopback tests), benches, launch lists.
O=gpurun_out/r2d
mkdir -p $O
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=40 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
for w in c0 c1 c2 c3 c4; do
  timeout 900 python bench.py --workload $w --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
KSEL='regex:estep|mstep|colsum|rowdot|list_kernel|bbox|zreduce|transform_sigma|sigma_final|spectral_rank'
CMD1="python bench.py --workload c1 --secondary none --steps 5 --warmup 3 --no-cpu --e2e-calls 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KSEL" -c 120 --csv --log-file $O/launches_c1.csv $CMD1 > $O/ncu_launch_c1.log 2>&1
CMD4="python bench.py --workload c4 --secondary none --steps 100 --warmup 3 --no-cpu --e2e-calls 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KSEL" -c 2000 --csv --log-file $O/launches_c4.csv $CMD4 > $O/ncu_launch_c4.log 2>&1
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED|Error" $O/pytest_gpu.txt | head -20; tail -1 $O/smoke.txt
for f in $O/bench_*.json; do echo "== $f"; cut -c1-200 $f; done
