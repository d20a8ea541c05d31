#!/bin/bash
# vertex sub-parts (L2 blocking at P=1) and the accumulated update rule, C3 / c3u / C2
for k in 4 16 64 256; do timeout 300 python tools/probe.py c3 2 $k 2>&1 | tail -1; done
for k in 4 64; do timeout 300 python tools/probe.py c3u 2 $k 2>&1 | tail -1; done
for k in 4 64; do timeout 300 python tools/probe.py c2 2 $k 2>&1 | tail -1; done
timeout 300 python tools/probe.py c3 2 4 1 2>&1 | tail -1
timeout 300 python tools/probe.py c3u 2 4 1 2>&1 | tail -1
