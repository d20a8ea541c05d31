#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "deterministic_shapes or c1" 2>&1 | tail -2
for v in "NE_SGNS_G8=0" "NE_SGNS_G8=1 NE_SGNS_MINB=2" "NE_SGNS_G8=1 NE_SGNS_MINB=1"; do echo "$v"; env $v timeout 600 python tools/probe.py c4 2 2>&1 | tail -1; done
