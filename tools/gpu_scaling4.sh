#!/bin/bash
# Final 4-GPU box: full GPU test suite (single + multi-GPU), then C3 / C4 scaling at N = 4, 2, 1
# (bench contract: W >= 3; every run under its own timeout).
mkdir -p gpurun_out/scale
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/scale/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/scale/tests.log; tail -2 gpurun_out/scale/tests.log
summ() { python -c "
import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1])
print('$1', d['n_gpus'], round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, 'e2e', round(d['e2e']['value']/1e6), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$1 failed"; }
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/scale/c3_n$N.json 2> gpurun_out/scale/c3_n$N.err; summ gpurun_out/scale/c3_n$N.json
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/scale/c3_n1.json 2> gpurun_out/scale/c3_n1.err; summ gpurun_out/scale/c3_n1.json
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/scale/c4_n$N.json 2> gpurun_out/scale/c4_n$N.err; summ gpurun_out/scale/c4_n$N.json
done
timeout 900 python bench.py --workload c4 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/scale/c4_n1.json 2> gpurun_out/scale/c4_n1.err; summ gpurun_out/scale/c4_n1.json
