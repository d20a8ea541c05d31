#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for cfg in "16 2" "16 3" "32 3"; do set -- $cfg; echo "LANES=$1 MINB=$2"; NE_SGNS_LANES=$1 NE_SGNS_MINB=$2 python tools/probe.py c3 2 2>&1 | tail -1; NE_SGNS_LANES=$1 NE_SGNS_MINB=$2 python tools/probe.py c2 2 2>&1 | tail -1; done
python tools/hogwild_diag.py 2>&1 | tail -7
