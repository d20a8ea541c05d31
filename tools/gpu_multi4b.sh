#!/bin/bash
python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2
for N in 4 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/c3_n$N.json 2> gpurun_out/c3_n$N.err; tail -1 gpurun_out/c3_n$N.err; cut -c1-400 gpurun_out/c3_n$N.json
done
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c3_n1.json 2>/dev/null; cut -c1-300 gpurun_out/c3_n1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 4 --workload c4 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/c4_n4.json 2> gpurun_out/c4_n4.err; tail -2 gpurun_out/c4_n4.err; cat gpurun_out/c4_n4.json
python bench.py --workload c4 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; tail -2 gpurun_out/c4_n1.err; cat gpurun_out/c4_n1.json
