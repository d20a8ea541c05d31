#!/bin/bash
# bf16 rows (NEXT-4): parity tests, then bench C3 f32 and bf16 back to back (twice, alternating)
mkdir -p gpurun_out/bf
timeout 1500 python -m pytest tests/test_gpu_bf16.py -q -s -k "matching or epoch or auc" > gpurun_out/bf/tests_bf16.log 2>&1; echo "rc=$?" >> gpurun_out/bf/tests_bf16.log
for i in; do
timeout 900 python bench.py --storage bf16 --no-cpu-baseline > gpurun_out/bf/bench_c3_bf16_$i.json 2> gpurun_out/bf/bench_c3_bf16_$i.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bf/bench_c3_f32_$i.json 2> gpurun_out/bf/bench_c3_f32_$i.err
done
grep -a "Frobenius\|passed\|failed\|rc=" gpurun_out/bf/tests_bf16.log | tail -12
for f in gpurun_out/bf/bench_c3_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6), round(d['ms_per_step'],1), {k:round(v,1) for k,v in d['phases_ms_per_step'].items()}, round(d['roofline']['achieved']), d['clocks'])"; done
