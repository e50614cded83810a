#!/bin/bash
O=gpurun_out/probe
mkdir -p $O
FCPD_CULL_PROBE=$P timeout 300 python tools/cull_trace.py c1 90 > $O/plain_p$P.json 2>&1 && \
FCPD_CULL_PROBE=$P timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"list_kernel|estep_row_kernel|estep_col_kernel" --launch-skip 320 --launch-count 16 --csv --log-file $O/ncu_list_p$P.csv python tools/cull_trace.py c1 90 > $O/ncu_p$P.log 2>&1
echo "exit $?"
grep -E "list_kernel|estep_row|estep_col" $O/ncu_list_p$P.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60,200- | head -20
