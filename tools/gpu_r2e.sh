#!/bin/bash
# Round-2 pass E: HMMA pass-2 prototype microbenchmark; culling re-check and
# row-dot prefetch benches.
O=gpurun_out/r2e
mkdir -p $O
./tools/pass2_hmma_bench > $O/pass2_hmma.txt 2>&1
./tools/loopbench > $O/loopbench.txt 2>&1
for w in c4 c3; do
  timeout 900 python bench.py --workload $w --secondary none --warmup 5 --no-cpu --e2e-calls 0 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --workload c4 --secondary none --steps 20 --warmup 5 --no-cpu --e2e-calls 0 > $O/bench_c4_20.json 2> $O/bench_c4_20.err
cat $O/pass2_hmma.txt
for f in $O/bench_*.json; do echo "== $f"; cut -c1-200 $f; done
