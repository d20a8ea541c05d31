#!/bin/bash
# full GPU suite; SGNS ncu --set full on C4 (fp32) and C3 (bf16 rows), reduced to CSV on the box
mkdir -p gpurun_out/re
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/re/tests.log 2>&1; echo "rc=$?" >> gpurun_out/re/tests.log; tail -3 gpurun_out/re/tests.log
for spec in "c4 0" "c3 1"; do
  set -- $spec; w=$1; st=$2
  PCMD="python tools/probe.py $w 1 4 0 $st"
  timeout 900 $PCMD > gpurun_out/re/probe_${w}_$st.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o /tmp/sg_${w}_$st $PCMD > gpurun_out/re/ncu_${w}_$st.log 2>&1
  ncu -i /tmp/sg_${w}_$st.ncu-rep --page raw --csv > gpurun_out/re/sgns_${w}_${st}_raw.csv 2>/dev/null
  tail -2 gpurun_out/re/probe_${w}_$st.log
done
