#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/probe.py c3 2 2>&1 | tail -1
