#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 250 > /tmp/clk.csv &
CP=$!
for w in c3 c2 c3u; do python tools/probe.py $w 3 2>&1 | tail -1; done
kill $CP; python - <<'PY'
import statistics
rows=[l.strip().split(',') for l in open('/tmp/clk.csv') if l.strip()]
sm=[float(r[0].split()[0]) for r in rows if 'MHz' in r[0]]
print('clock median MHz', statistics.median(sm), 'max', max(sm), 'power-cap active frac', sum('Active' in r[2] for r in rows)/len(rows))
PY
