bash tools/gpu.sh r4b \
  torchrun:4:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline,--transport,ipc \
  torchrun:2:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline,--transport,ipc \
  torchrun:4:--steps,5,--warmup,3,--e2e-steps,2,--transport,ipc \
  torchrun:2:--steps,5,--warmup,3,--e2e-steps,2,--transport,ipc \
  env:NE_PIPELINE=0 torchrun:4:--workload,c4,--steps,2,--warmup,2,--e2e-steps,1,--no-cpu-baseline,--transport,ipc env:NE_PIPELINE= \
  torchrun:4:--workload,c5,--steps,2,--warmup,2,--e2e-steps,1,--no-cpu-baseline,--transport,ipc \
  torchrun:4:--workload,c5,--steps,2,--warmup,2,--e2e-steps,1,--no-cpu-baseline
