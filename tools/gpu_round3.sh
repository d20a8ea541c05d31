#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -6
for t in 0 1; do echo "TMA=$t"; for w in c3 c2 c3u; do NE_SGNS_TMA=$t python tools/probe.py $w 2 2>&1 | tail -1; done; done
