#!/bin/bash
# Official round artefacts: bench (N=1), launch list of the same command, ncu full capture of SGNS on C3.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc; lscpu | grep "Model name"
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err; cat gpurun_out/bench_n1.json
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$BCMD > gpurun_out/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
PCMD="python tools/probe.py c3 1"
$PCMD > gpurun_out/probe_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o gpurun_out/sgns_c3_v3 $PCMD > gpurun_out/ncu_full_c3.log 2>&1
tail -2 gpurun_out/ncu_full_c3.log
PCMD="python tools/probe.py c3u 1"
$PCMD > gpurun_out/probe_c3u.log 2>&1 && \
  ncu --set full --clock-control none -k regex:sgns -s 1 -c 1 -o gpurun_out/sgns_c3u_v3 $PCMD > gpurun_out/ncu_full_c3u.log 2>&1
tail -2 gpurun_out/ncu_full_c3u.log
