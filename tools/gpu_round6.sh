#!/bin/bash
python -m pytest tests -m gpu -q -x -k "node2vec or reload" 2>&1 | tail -3
timeout 900 python tools/probe.py c4 2 2>&1 | tail -6
timeout 900 python tools/probe.py c5 2 2>&1 | tail -6
