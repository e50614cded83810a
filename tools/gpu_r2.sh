#!/bin/bash
# Centred-form guard study: parity logs and C2/C4 trajectories at R² limits.
O=gpurun_out/r2
mkdir -p $O
for r2 in 16 64 256; do
  rm -f $O/parity_$r2.jsonl
  FCPD_CENTRED_MAX_R2=$r2 FCPD_PARITY_LOG=$O/parity_$r2.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "estep_matches or c0_parity or c1_reduced or full_size or register_matches or culling" > $O/pytest_$r2.txt 2>&1
  echo "r2=$r2 $(tail -1 $O/pytest_$r2.txt)"
  for w in c2 c4; do FCPD_CENTRED_MAX_R2=$r2 python tools/cull_trace.py $w > $O/trace_${w}_$r2.json 2>/dev/null; done
done
