#!/bin/bash
python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python tools/hogwild_diag.py 2>&1 | tail -8
for add in 0 1; do python - <<PY
import sys; sys.path.insert(0,'.')
import synth
from paper_2005_13789_b200.engine import Engine
off,tgt = synth.workload_graph('c3')
for pm in (10**6, 100):
    e = Engine(dim=128, conflict_permille=pm, writeback=1-$add); e.load_graph(off,tgt)
    for ep in range(2): st = e.train_epoch(ep, 0.025)
    print('c3 add=$add permille', pm, 'kernel M samples/s %.1f' % (st['samples']/st['ms_train']/1e3), 'loss %.4f' % (st['loss_sum']/st['samples']/6), flush=True)
    e.close()
PY
done
python tools/hogwild_quality.py 1 2>&1 | tail -8
