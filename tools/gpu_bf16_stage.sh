#!/bin/bash
mkdir -p gpurun_out/bfs
timeout 1200 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_parity.py -q -k "bf16 or staged" > gpurun_out/bfs/tests.log 2>&1; echo "rc=$?" >> gpurun_out/bfs/tests.log
tail -4 gpurun_out/bfs/tests.log
