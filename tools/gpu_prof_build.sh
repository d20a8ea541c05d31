#!/bin/bash
mkdir -p gpurun_out/pb
CMD="python tools/probe_build.py c3 1"
timeout 300 $CMD > gpurun_out/pb/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pairs_walk|bucket_scatter" -s 2 -c 2 -o /tmp/pb $CMD > gpurun_out/pb/ncu.log 2>&1
ncu -i /tmp/pb.ncu-rep --page raw --csv > gpurun_out/pb/raw.csv 2>/dev/null
ncu -i /tmp/pb.ncu-rep --page source --csv --print-source sass > gpurun_out/pb/source.csv 2>/dev/null
tail -2 gpurun_out/pb/ncu.log
