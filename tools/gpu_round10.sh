#!/bin/bash
mkdir -p gpurun_out/prof10
CMD="python tools/probe_build.py c4 4"
$CMD > gpurun_out/prof10/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/prof10/build_c4_p4.csv $CMD > gpurun_out/prof10/ncu.log 2>&1
tail -2 gpurun_out/prof10/plain.log
