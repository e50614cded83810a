#!/bin/bash
# Round-2 pass F: 2-step top-K setup with the device RNG (accuracy tests +
# setup times), fp32-batched row-dot z pass.
O=gpurun_out/r2f
mkdir -p $O
rm -f $O/parity.jsonl
FCPD_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -q -m gpu -rA --durations=20 > $O/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.txt
for w in c4 c3 c2; do
  timeout 900 python bench.py --workload $w --secondary none --warmup 5 --no-cpu --e2e-calls 1 > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/pytest_gpu.txt; grep -E "^FAILED|Error" $O/pytest_gpu.txt | head -20
for f in $O/bench_*.json; do echo "== $f"; cut -c1-200 $f; done
