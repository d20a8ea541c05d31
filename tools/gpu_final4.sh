#!/bin/bash
# final code, 4-GPU box: the complete GPU suite (single-GPU parity, bf16, torchrun 2/4-rank ring)
mkdir -p gpurun_out/f4
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/f4/tests.log 2>&1; echo "rc=$?" >> gpurun_out/f4/tests.log
tail -3 gpurun_out/f4/tests.log
