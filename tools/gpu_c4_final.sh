#!/bin/bash
# final code, one 4-GPU box: C4 at N = 4, 2, 1 back to back (W = 3)
mkdir -p gpurun_out/c4f
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2993$N bench.py --gpus $N --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/c4f/c4_n$N.json 2> gpurun_out/c4f/c4_n$N.err; summ gpurun_out/c4f/c4_n$N.json
done
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/c4f/c4_n1.json 2> gpurun_out/c4f/c4_n1.err; summ gpurun_out/c4f/c4_n1.json
