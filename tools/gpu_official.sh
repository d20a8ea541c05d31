#!/bin/bash
# Official round artefacts (single GPU): bench line, launch list of the same command shape,
# ncu --set full of the SGNS kernel on C3 and on the uniform control (reduced to CSV on the box).
mkdir -p gpurun_out/off
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
nproc; lscpu | grep "Model name"
timeout 900 python bench.py > gpurun_out/off/bench_n1.json 2> gpurun_out/off/bench_n1.err; tail -2 gpurun_out/off/bench_n1.err
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/off/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/off/launches.csv $BCMD > gpurun_out/off/ncu_launches.log 2>&1
for w in c3 c3u; do
  PCMD="python tools/probe.py $w 1"
  timeout 600 $PCMD > gpurun_out/off/probe_$w.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o /tmp/sgns_$w $PCMD > gpurun_out/off/ncu_full_$w.log 2>&1
  ncu -i /tmp/sgns_$w.ncu-rep --page raw --csv > gpurun_out/off/sgns_${w}_raw.csv 2>/dev/null
  ncu -i /tmp/sgns_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/off/sgns_${w}_source.csv 2>/dev/null
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/off/ref_n1.json 2> gpurun_out/off/ref_n1.err; tail -1 gpurun_out/off/ref_n1.err
du -sh gpurun_out/off
