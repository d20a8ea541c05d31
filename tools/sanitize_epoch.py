"""compute-sanitizer target: one deterministic and one Hogwild epoch of a
small R-MAT graph through the C ABI (walk, pool build -- keyed radix path and
direct scatter --, SGNS), checked against the oracle so a sanitizer run also
shows the results stayed correct.  Run under
`compute-sanitizer --tool memcheck|racecheck python tools/sanitize_epoch.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2005_13789_b200.engine import Engine  # noqa: E402

off, tgt = synth.rmat_graph(3000, 20000, 5)
n = len(off) - 1
kw = dict(dim=64, negatives=5, walk_len=12, window=3, walks_per_node=1, episodes=2, subparts=3, seed=42)
for direct in ("0", "1"):
    os.environ["NE_POOL_DIRECT"] = direct
    eng = Engine(deterministic=True, **kw)
    eng.load_graph(off, tgt)
    st = eng.train_epoch(0, 0.025)
    V = oracle.init_vertex(n, 64, 42)
    Cm = np.zeros_like(V)
    ns, _ = oracle.train_epoch(oracle.Config(parts=1, **kw), off, tgt, V, Cm, 0, 0.025)
    dv = float(np.abs(eng.embeddings(0) - V).max())
    assert st["samples"] == ns and dv <= 1e-4, (st["samples"], ns, dv)
    eng.close()
    eng = Engine(deterministic=False, **kw)
    eng.load_graph(off, tgt)
    st = eng.train_epoch(0, 0.025)
    assert np.isfinite(eng.embeddings(0)).all()
    eng.close()
    print(f"direct={direct}: deterministic max|dV| {dv:.2e}, hogwild samples {st['samples']}", flush=True)
print("sanitize_epoch ok")
