#!/bin/bash
# re-entry check on a fresh box: GPU suite, smoke(), default N=1 bench
mkdir -p gpurun_out/rx
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/rx/tests.log 2>&1; echo "rc=$?" >> gpurun_out/rx/tests.log; tail -3 gpurun_out/rx/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rx/smoke.log 2>&1; tail -2 gpurun_out/rx/smoke.log
timeout 600 python bench.py > gpurun_out/rx/bench_n1.json 2> gpurun_out/rx/bench_n1.err; tail -c 600 gpurun_out/rx/bench_n1.json
