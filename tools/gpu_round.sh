#!/bin/bash
# One GPU session: tests, bench, launch list, ncu capture of the SGNS kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -m pytest tests -m gpu -q 2>&1 | tail -15
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -3 gpurun_out/bench_n1.err; cat gpurun_out/bench_n1.json
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$BCMD > gpurun_out/bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
PCMD="python tools/probe.py c2 1"
$PCMD > gpurun_out/probe_c2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sgns -s 1 -c 1 -o gpurun_out/sgns_c2 $PCMD > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
