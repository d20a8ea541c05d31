#!/bin/bash
# Final single-GPU pass: smoke, full GPU suite, official N = 1 bench + reference arm + launch list,
# and bf16 occupancy knobs (probe, kernel-only samples/s).
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv,noheader
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log; tail -2 gpurun_out/fin/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fin/tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin/tests.log; tail -2 gpurun_out/fin/tests.log
timeout 900 python bench.py > gpurun_out/fin/bench_n1.json 2> gpurun_out/fin/bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/ref_n1.json 2> gpurun_out/fin/ref_n1.err
BCMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/fin/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches.csv $BCMD > gpurun_out/fin/ncu_launches.log 2>&1
for knob in "" "NE_SGNS_MINB=3" "NE_SGNS_LANES=32"; do
  env $knob timeout 300 python tools/probe.py c3 2 4 0 1 2>&1 | tail -1 | sed "s/^/bf16 [$knob] /"
done
python -c "
import json
for f in ['gpurun_out/fin/bench_n1.json','gpurun_out/fin/ref_n1.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d.get('value'), d.get('ms_per_step'), d.get('clocks'))
    except Exception as e: print(f, 'failed', e)"
