#!/bin/bash
# Round-2 first GPU pass: the GPU suite (with the new full-size parity file)
# and the C4 / C1 bench lines of the current build.
O=gpurun_out/r2a
mkdir -p $O
rm -f $O/parity.jsonl
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=25 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
for w in c4 c1; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED|Error" $O/pytest_gpu.txt | head -20
for f in $O/bench_*.json; do echo "== $f"; cut -c1-300 $f; done
