"""Link-prediction AUC at YouTube scale (C2-shaped, 1% held-out edges):
deterministic (= oracle order, parity-checked) vs Hogwild variants."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import oracle, synth
from paper_2005_13789_b200.engine import Engine

w = synth.CONFIGS["c2"]
t = time.time()
u, v = synth.rmat_edges(w.n, w.m, w.graph_seed)
off, tgt, test = synth.split_edges(w.n, u, v, 0.01, 7)
neg = synth.negative_pairs(w.n, u, v, len(test), 8)
print(f"split {len(test)} test edges, {time.time()-t:.1f}s", flush=True)
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for det, pm, add in [(False, 10**6, 0), (False, 10**6, 1), (False, 100, 0), (False, 100, 1), (True, 0, 0)]:
    eng = Engine(dim=128, deterministic=det, conflict_permille=pm, writeback=0 if add else 1)
    eng.load_graph(off, tgt)
    t = time.time()
    for ep in range(epochs):
        st = eng.train_epoch(ep, 0.025)
    Vg, Cg = eng.embeddings(0), eng.embeddings(1)
    a = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
    print(f"det={det} permille={pm} add={add} epochs={epochs} auc={a:.4f} last-epoch loss/sample="
          f"{st['loss_sum']/st['samples']/6:.4f} train {st['ms_train']:.0f} ms wall {time.time()-t:.1f}s", flush=True)
    eng.close()
