#!/bin/bash
# Round-2 pass K: DMMA Φ·V kernel — top-K parity, setup times vs the DFMA
# kernel, ncu of one product at C2.
O=gpurun_out/r2k
mkdir -p $O
./tools/exp_nonpos_test > $O/exp_test.txt 2>&1; cat $O/exp_test.txt
export FCPD_TOPK_LOG=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_parity_full.py -q -m gpu -k "topk or lowrank" -s > $O/pytest_topk.txt 2>&1
echo "pytest exit $?" >> $O/pytest_topk.txt
for w in c2 c3 c4; do
  timeout 600 python tools/run_topk.py $w > $O/topk_$w.txt 2>&1
  FCPD_GRAM_DFMA=1 timeout 600 python tools/run_topk.py $w > $O/topk_dfma_$w.txt 2>&1
done
unset FCPD_TOPK_LOG
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_dmma -c 1 -o $O/gram_dmma_c2 python tools/run_topk.py c2 > $O/ncu_gram.log 2>&1
tail -3 $O/pytest_topk.txt; grep -E "^FAILED|Error|topk:" $O/pytest_topk.txt | head -40; cat $O/topk_*.txt; tail -2 $O/ncu_gram.log
