#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for P in 1 4 8; do python tools/probe_build.py c3 $P 2>&1 | tail -1; done
python tools/probe.py c3 2 2>&1 | tail -1
python tools/probe_build.py c4 8 2>&1 | tail -1
