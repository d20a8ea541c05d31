#!/bin/bash
# ncu artefacts, reduced to CSV on the box (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out/prof
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$BCMD > gpurun_out/prof/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv $BCMD > gpurun_out/prof/ncu_launches.log 2>&1
for w in c3 c3u; do
  PCMD="python tools/probe.py $w 1"
  $PCMD > gpurun_out/prof/probe_$w.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o /tmp/sgns_$w $PCMD > gpurun_out/prof/ncu_full_$w.log 2>&1
  ncu -i /tmp/sgns_$w.ncu-rep --page raw --csv > gpurun_out/prof/sgns_${w}_raw.csv 2>/dev/null
  ncu -i /tmp/sgns_$w.ncu-rep --page details --csv > gpurun_out/prof/sgns_${w}_details.csv 2>/dev/null
  ncu -i /tmp/sgns_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/sgns_${w}_source.csv 2>/dev/null
  ls -la /tmp/sgns_$w.ncu-rep
done
du -sh gpurun_out
