#!/bin/bash
mkdir -p gpurun_out/prof8
CMD="python tools/probe_build.py c3 8"
$CMD > gpurun_out/prof8/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"bucket_scatter|pairs_walk|bucket_count" -s 3 -c 3 -o /tmp/build8 $CMD > gpurun_out/prof8/ncu.log 2>&1
ncu -i /tmp/build8.ncu-rep --page raw --csv > gpurun_out/prof8/raw.csv 2>/dev/null
ncu -i /tmp/build8.ncu-rep --page source --csv --print-source sass > gpurun_out/prof8/source.csv 2>/dev/null
ls -la /tmp/build8.ncu-rep; du -sh gpurun_out/prof8
python tools/probe.py c5 2 2>&1 | tail -2
