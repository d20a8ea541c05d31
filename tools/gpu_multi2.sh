#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -3
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 3 --warmup 2 > gpurun_out/c3_n2b.json 2> gpurun_out/c3_n2b.err; tail -1 gpurun_out/c3_n2b.err; python -c "
import json; d=json.loads(open('gpurun_out/c3_n2b.json').read().strip().splitlines()[-1])
print('c3 n2', round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()})"
