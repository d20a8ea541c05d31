#!/bin/bash
nvidia-smi -L
python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -4
for N in 4 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 3 --warmup 2 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; tail -2 gpurun_out/bench_n$N.err; cat gpurun_out/bench_n$N.json
done
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_n1_short.json 2>/dev/null; cat gpurun_out/bench_n1_short.json
