#!/bin/bash
# full GPU suite + N=1 bench + launch list of the bench command shape
mkdir -p gpurun_out/chk
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/chk/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/chk/tests.log
timeout 900 python bench.py > gpurun_out/chk/bench_n1.json 2> gpurun_out/chk/bench_n1.err
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/chk/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chk/launches.csv $BCMD > gpurun_out/chk/ncu_launches.log 2>&1
tail -3 gpurun_out/chk/tests.log; cat gpurun_out/chk/bench_n1.json
