#!/bin/bash
mkdir -p gpurun_out/dbg
for m in 0 1 2 3; do
  for d in 0 1; do
    NE_POOL_DBG=$m NE_POOL_DIRECT=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pairs_walk" --csv --log-file gpurun_out/dbg/m${m}_d${d}.csv python tools/probe_build.py c3 1 > gpurun_out/dbg/m${m}_d${d}.log 2>&1
    echo "mode $m direct $d: $(grep pairs_walk gpurun_out/dbg/m${m}_d${d}.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
  done
done
