#!/bin/bash
mkdir -p gpurun_out/p8
timeout 300 python tools/probe_build.py c3 8 > gpurun_out/p8/plain.log 2>&1; tail -2 gpurun_out/p8/plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"walk|pairs|bucket|window|count|scan|radix" --csv --log-file gpurun_out/p8/launches.csv python tools/probe_build.py c3 8 > gpurun_out/p8/ncu.log 2>&1
python tools/ncu_summary.py launches gpurun_out/p8/launches.csv | head -14
