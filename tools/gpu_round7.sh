#!/bin/bash
mkdir -p gpurun_out/prof7
for P in 1 4 8; do python tools/probe_build.py c3 $P 2>&1 | tail -1; done
CMD="python tools/probe_build.py c3 8"
$CMD > gpurun_out/prof7/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof7/build_p8.csv $CMD > gpurun_out/prof7/ncu.log 2>&1
CMD="python tools/probe_build.py c3 1"
$CMD > gpurun_out/prof7/plain1.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof7/build_p1.csv $CMD > gpurun_out/prof7/ncu1.log 2>&1
cuobjdump -res-usage paper_2005_13789_b200/libne_b200.so 2>/dev/null | grep -A1 "sgns_kernelILi32ELi2ELi5ELi3ELb1" | tail -1
