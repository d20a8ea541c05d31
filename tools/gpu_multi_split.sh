#!/bin/bash
# walk all-gather on a split communicator: multi-GPU parity, then C4 / C3 at N = 4 (each under its own timeout)
mkdir -p gpurun_out/ms
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/ms/tests.log 2>&1; echo "rc=$?" >> gpurun_out/ms/tests.log; tail -2 gpurun_out/ms/tests.log
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29734 bench.py --gpus 4 --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/ms/c4_n4.json 2> gpurun_out/ms/c4_n4.err; summ gpurun_out/ms/c4_n4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29714 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/ms/c3_n4.json 2> gpurun_out/ms/c3_n4.err; summ gpurun_out/ms/c3_n4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/ms/c3_n2.json 2> gpurun_out/ms/c3_n2.err; summ gpurun_out/ms/c3_n2.json
