"""AUC of Hogwild training vs concurrency and write-back mode (planted partition, n=2000)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle, synth
from paper_2005_13789_b200.engine import Engine

n = 2000
u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
neg = synth.negative_pairs(n, u, v, len(test), 8)
kw = dict(dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1)
for det, pm, add in [(True, 0, 0), (False, 100, 0), (False, 100, 1), (False, 300, 1), (False, 1000, 1),
                     (False, 10**6, 1), (False, 10**6, 0)]:
    eng = Engine(deterministic=det, conflict_permille=pm, writeback=0 if add else 1, **kw)
    eng.load_graph(off, tgt)
    losses = []
    for ep in range(2):
        st = eng.train_epoch(ep, 0.05)
        losses.append(round(st["loss_sum"] / st["samples"], 3))
    Vg, Cg = eng.embeddings(0), eng.embeddings(1)
    a = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
    print(f"det={det} permille={pm} add={add} auc={a:.4f} loss/sample={losses}", flush=True)
    eng.close()
