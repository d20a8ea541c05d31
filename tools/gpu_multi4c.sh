#!/bin/bash
run() { # name, env...
  name=$1; shift
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 4 --workload c4 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$name.json').read().strip().splitlines()[-1])
print('$name', round(d['value']/1e6), 'M/s', round(d['ms_per_step'],1), 'ms', {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, d['clocks']['sm_mhz'])" 2>/dev/null || tail -3 gpurun_out/ab_$name.err
}
run res2 NE_RING_RESERVE_SMS=2
run res0 NE_RING_RESERVE_SMS=0
run res4 NE_RING_RESERVE_SMS=4
run ce0 NE_RING_RESERVE_SMS=0 NCCL_P2P_USE_CUDA_MEMCPY=1
python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2
