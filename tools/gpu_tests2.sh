#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
cat > /tmp/stage_probe.py <<'PY'
import sys, time; sys.path.insert(0, ".")
import synth, torch
from paper_2005_13789_b200.engine import Engine
name = sys.argv[1]; w = synth.CONFIGS[name]
off, tgt = synth.workload_graph(name, device="cuda")
for staging, k in [(0, 4), (1, 16)]:
    eng = Engine(dim=w.dim, episodes=w.episodes, subparts=k, staging=staging)
    eng.load_graph(off, tgt)
    for ep in range(2):
        t = time.time(); st = eng.train_epoch(ep, 0.025); wall = time.time() - t
    print(f"{name} staging={staging} k={k}: epoch wall {wall:.3f}s train {st['ms_train']:.0f} ms samples {st['samples']} "
          f"-> {st['samples']/wall/1e6:.0f} M/s step; free {torch.cuda.mem_get_info()[0]/1e9:.1f} GB", flush=True)
    eng.close(); torch.cuda.empty_cache()
PY
timeout 400 python /tmp/stage_probe.py c3
timeout 600 python /tmp/stage_probe.py c4
