#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for am in 0 1; do echo "AMORT=$am"; NE_SGNS_AMORT=$am python tools/probe.py c3 2 2>&1 | tail -1; NE_SGNS_AMORT=$am python tools/probe.py c2 2 2>&1 | tail -1; NE_SGNS_AMORT=$am python tools/probe.py c3u 2 2>&1 | tail -1; done
PCMD="python tools/probe.py c3 1"
$PCMD > gpurun_out/probe_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o gpurun_out/sgns_c3_v2 $PCMD > gpurun_out/ncu_full_c3.log 2>&1
tail -2 gpurun_out/ncu_full_c3.log
