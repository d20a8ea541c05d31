#!/bin/bash
# sliced CSR load (1/P per rank over PCIe + NVLink all-gather): multi-GPU parity, then C3 at N = 4, 2 (e2e)
mkdir -p gpurun_out/sl
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/sl/tests.log 2>&1; echo "rc=$?" >> gpurun_out/sl/tests.log; tail -2 gpurun_out/sl/tests.log
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2978$N bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/sl/c3_n$N.json 2> gpurun_out/sl/c3_n$N.err; summ gpurun_out/sl/c3_n$N.json
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29794 bench.py --gpus 4 --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/sl/c4_n4.json 2> gpurun_out/sl/c4_n4.err; summ gpurun_out/sl/c4_n4.json
