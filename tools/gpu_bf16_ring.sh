#!/bin/bash
# bf16 rows over the NCCL ring: multi-GPU parity (2, 4 ranks), emulation, C3 bf16 at N = 4
mkdir -p gpurun_out/bfr
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_bf16.py -q -k "bf16" -s > gpurun_out/bfr/tests.log 2>&1; echo "rc=$?" >> gpurun_out/bfr/tests.log
grep -a "MULTI\|passed\|failed\|rc=" gpurun_out/bfr/tests.log | tail -12
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29744 bench.py --gpus 4 --steps 3 --warmup 3 --storage bf16 > gpurun_out/bfr/c3bf_n4.json 2> gpurun_out/bfr/c3bf_n4.err
python -c "
import json; d=json.loads(open('gpurun_out/bfr/c3bf_n4.json').read().strip().splitlines()[-1]); print('c3 bf16 n4', round(d['value']/1e6), round(d['ms_per_step'],1), d['phases_ms_per_step'], d['clocks'])" || tail -5 gpurun_out/bfr/c3bf_n4.err
