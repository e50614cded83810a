#!/bin/bash
# Precision/speed study of the E-step pass-2 fp32 run length (FCPD_FLUSH2):
# parity tests + bench lines.  FLUSHES="256 64 32", WORKLOADS="c1 c2".
for f in ${FLUSHES:-256 64 32}; do
  rm -f gpurun_out/p.jsonl
  FCPD_FLUSH2=$f FCPD_PARITY_LOG=gpurun_out/p.jsonl timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c1_reduced or c0_parity" 2>&1 | tail -1
  echo "flush2 $f"; cut -c1-110 gpurun_out/p.jsonl
  for w in ${WORKLOADS:-c1}; do
  FCPD_FLUSH2=$f timeout 300 python bench.py --workload $w --no-cpu --e2e-calls 0 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w it/s', round(d['value'],1), {k: round(v,4) for k,v in d['phase_ms'].items() if k.startswith('estep')})"
  done
done
