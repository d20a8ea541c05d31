#!/bin/bash
# bench lines for the other BASELINE configs: C5 (node2vec q=0.5, d=256) at N = 4 and 1, C2 at N = 1
mkdir -p gpurun_out/c25
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'alg', round(d['roofline']['achieved']), 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29764 bench.py --gpus 4 --workload c5 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/c25/c5_n4.json 2> gpurun_out/c25/c5_n4.err; summ gpurun_out/c25/c5_n4.json
timeout 1200 python bench.py --workload c5 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/c25/c5_n1.json 2> gpurun_out/c25/c5_n1.err; summ gpurun_out/c25/c5_n1.json
timeout 900 python bench.py --workload c2 > gpurun_out/c25/c2_n1.json 2> gpurun_out/c25/c2_n1.err; summ gpurun_out/c25/c2_n1.json
tail -3 gpurun_out/c25/c5_n1.err
