bash tools/gpu.sh r4a info "tests:multi or ipc" \
  torchrun:4:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline \
  torchrun:2:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline \
  bench:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline \
  torchrun:4:--workload,c4,--episodes,16,--steps,2,--warmup,3,--e2e-steps,1,--no-cpu-baseline \
  torchrun:4:--workload,c4,--episodes,16,--steps,2,--warmup,3,--e2e-steps,1,--no-cpu-baseline,--transport,ipc \
  torchrun:4:--workload,c4,--steps,3,--warmup,3,--e2e-steps,1,--no-cpu-baseline,--groups,2 \
  torchrun:4:--steps,5,--warmup,3,--e2e-steps,2 torchrun:2:--steps,5,--warmup,3,--e2e-steps,2
