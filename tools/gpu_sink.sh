#!/bin/bash
# pool build: parity + full ncu of pairs_walk and a radix pass
mkdir -p gpurun_out/sink
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "pool or walk or det or c2 or ring" > gpurun_out/sink/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sink/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pairs_walk|radix" -s 2 -c 2 -o /tmp/pw python tools/probe_build.py c3 1 > gpurun_out/sink/ncu_full.log 2>&1
ncu -i /tmp/pw.ncu-rep --page raw --csv > gpurun_out/sink/pw_raw.csv 2>/dev/null
ncu -i /tmp/pw.ncu-rep --page source --csv --print-source sass > gpurun_out/sink/pw_source.csv 2>/dev/null
tail -3 gpurun_out/sink/tests.log
