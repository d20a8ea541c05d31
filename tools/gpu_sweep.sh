#!/bin/bash
python tools/hogwild_diag.py 2>&1 | tail -12
for m in 2 3 4; do echo "MINB=$m"; NE_SGNS_MINB=$m python tools/probe.py c3 2 2>&1 | tail -2; done
NE_SGNS_MINB=3 python tools/probe.py c2 2 2>&1 | tail -1
