#!/bin/bash
mkdir -p gpurun_out/last
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last/smoke.log; tail -2 gpurun_out/last/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/last/tests.log 2>&1; echo "rc=$?" >> gpurun_out/last/tests.log; tail -2 gpurun_out/last/tests.log
