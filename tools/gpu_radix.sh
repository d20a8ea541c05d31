#!/bin/bash
mkdir -p gpurun_out/rx
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "radix or sinks or grow" > gpurun_out/rx/tests.log 2>&1; echo "rc=$?" >> gpurun_out/rx/tests.log
tail -3 gpurun_out/rx/tests.log
