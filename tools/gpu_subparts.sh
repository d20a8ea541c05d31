#!/bin/bash
for k in 4 16 64 256; do python tools/probe.py c3 2 $k 2>&1 | tail -1; done
for k in 4 64; do python tools/probe.py c3u 2 $k 2>&1 | tail -1; done
for k in 4 64; do python tools/probe.py c2 2 $k 2>&1 | tail -1; done
