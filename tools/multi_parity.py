"""torchrun worker: P-rank training over the real NCCL ring on P GPUs, compared
with the oracle's P-part epochs (run by rank 0): deterministic mode within 1e-4
(max-abs), Hogwild mode by link-prediction AUC within 0.01 of the oracle's
(SURVEY 8(c) gate: C1, 10% held-out edges, 5 epochs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import oracle
import synth
from paper_2005_13789_b200 import ne
from paper_2005_13789_b200.engine import Engine


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    mode = sys.argv[1] if len(sys.argv) > 1 else "det"
    kind = sys.argv[2] if len(sys.argv) > 2 else "deepwalk"
    extra = {"deepwalk": {}, "node2vec": dict(p=0.5, q=2.0), "line": dict(walk_len=0, window=0),
             "groups2": dict(groups=2),  # NEXT-3 two-level ring: two groups of world/2 ranks
             "ipc": dict(transport=ne.NE_TRANSPORT_IPC),  # copy-engine ring over CUDA IPC (+ NCCL pool build)
             "staged": dict(staging=1, stage_window=2),   # NEXT-2 with the ring: host-staged parts, windows of 2
             # NEXT-4 bf16 rows over the ring, on a perfect matching (rows stored ~1+K times, the
             # element-wise bar of tests/test_gpu_bf16.py)
             "bf16": dict(walk_len=1, window=1, storage=1)}[kind]
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [ne.ne_get_nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    test = neg = None
    if kind == "bf16":
        u = np.arange(0, 20000, 2, dtype=np.int64)
        off, tgt = synth.csr_from_undirected(20000, u, u + 1)
    elif mode == "hogwild":
        w = synth.CONFIGS["c1"]
        u, v = synth.rmat_edges(w.n, w.m, w.graph_seed)
        off, tgt, test = synth.split_edges(w.n, u, v, 0.1, synth.EVAL_SEED)
        neg = synth.negative_pairs(w.n, u, v, len(test), synth.EVAL_SEED + 1)
    else:
        off, tgt = synth.workload_graph("c1")
    n = len(off) - 1
    epochs = 5 if mode == "hogwild" else 2
    eng = Engine(dim=128, deterministic=(mode == "det"), device=local, rank=rank, world=world,
                 nccl_id=obj[0], episodes=2, **extra)
    def all_gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    eng.load_graph(off, tgt, all_gather=all_gather)
    a, b = eng.part
    # the vertex rows stream out as their sub-parts come home (fp32 rows in HBM)
    exp = torch.full((b - a, 128), float("nan")).pin_memory() if kind not in ("staged", "bf16") else None
    if exp is not None:
        eng.export_vertex_on_train(exp)
    stats = [eng.train_epoch(ep, 0.025) for ep in range(epochs)]
    V, Cm = eng.embeddings(0), eng.embeddings(1)
    if exp is not None:
        assert np.array_equal(exp.numpy(), V), "exported vertex rows differ from ne_get_embeddings"
    parts = [None] * world
    dist.all_gather_object(parts, (a, b, V, Cm, stats))
    if rank == 0:
        base = dict(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=2,
                    subparts=4, parts=world, seed=42)
        base.update({k: v for k, v in extra.items() if k not in ("transport", "staging", "stage_window")})
        if kind == "staged":
            base["window_slots"] = 2
        cfg = oracle.Config(**base)
        Vr = oracle.init_vertex(n, 128, 42)
        if kind == "bf16":
            Vr = oracle.round_bf16(Vr)
        Cr = np.zeros_like(Vr)
        ns = 0
        for ep in range(epochs):
            ns += oracle.train_epoch(cfg, off, tgt, Vr, Cr, ep, 0.025)[0]
        got_ns = sum(st["samples"] for p in parts for st in p[4])
        assert got_ns == ns, (got_ns, ns)
        dv = max(np.abs(p[2] - Vr[p[0]:p[1]]).max() for p in parts)
        dc = max(np.abs(p[3] - Cr[p[0]:p[1]]).max() for p in parts)
        print(f"MULTI {mode} {kind} world={world} samples={ns} max|dV|={dv:.3e} max|dC|={dc:.3e}", flush=True)
        if mode == "det" and kind == "bf16":
            for i, R in ((2, Vr), (3, Cr)):
                got = np.concatenate([p[i] for p in parts])
                ref = np.concatenate([R[p[0]:p[1]] for p in parts])
                ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.maximum(np.abs(got), np.abs(ref)), 2.0**-14))) - 7)
                same, err = np.mean(got == ref), float((np.abs(got.astype(np.float64) - ref) / ulp).max())
                print(f"MULTI bf16 matrix {i - 2}: identical {same:.5f}, max {err:.1f} ulp", flush=True)
                assert same >= 0.99 and err <= 2.0 + 5, (same, err)
        elif mode == "det":
            assert dv <= 1e-4 and dc <= 1e-4, (dv, dc)
        else:  # Hogwild: the AUC gate
            Vg = np.concatenate([p[2] for p in parts])
            Cg = np.concatenate([p[3] for p in parts])
            a_ref = oracle.auc(oracle.score_pairs(Vr, Cr, test), oracle.score_pairs(Vr, Cr, neg))
            a_gpu = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
            print(f"MULTI hogwild AUC world={world}: gpu {a_gpu:.4f} oracle {a_ref:.4f}", flush=True)
            assert np.isfinite(Vg).all() and np.isfinite(Cg).all()
            assert abs(a_gpu - a_ref) <= 0.01, (a_gpu, a_ref)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
