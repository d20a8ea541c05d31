#!/bin/bash
# final code, one 4-GPU box: C3 at N = 4, 2, 1 back to back (W = 3, 5 timed steps)
mkdir -p gpurun_out/sf
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N bench.py --gpus $N > gpurun_out/sf/c3_n$N.json 2> gpurun_out/sf/c3_n$N.err; summ gpurun_out/sf/c3_n$N.json
done
timeout 600 python bench.py > gpurun_out/sf/c3_n1.json 2> gpurun_out/sf/c3_n1.err; summ gpurun_out/sf/c3_n1.json
