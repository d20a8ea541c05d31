#!/bin/bash
# NCCL CTA cap vs ring interference: C4 at 16 episodes, N = 4 (each under its own timeout)
mkdir -p gpurun_out/ctas
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'clk', d['clocks']['sm_mhz'])" 2>/dev/null || echo "$1 failed"; }
for c in default 2 8; do
  if [ $c = default ]; then E=""; else E="NCCL_MAX_CTAS=$c"; fi
  env $E timeout 700 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2990${#c} bench.py --gpus 4 --workload c4 --episodes 16 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/ctas/c4e16_$c.json 2> gpurun_out/ctas/c4e16_$c.err; summ gpurun_out/ctas/c4e16_$c.json
done
