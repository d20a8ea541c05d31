"""torchrun worker (gloo for the host bootstrap): P-rank training whose ring
moves vertex sub-parts with copy-engine pushes over CUDA IPC
(NE_TRANSPORT_IPC), no NCCL.  Ranks share GPUs round-robin, so the test runs
on a single-GPU box too (two or three processes on one device).  Rank 0
compares with the oracle's P-part epochs: deterministic mode within 1e-4,
Hogwild mode by held-out AUC within 0.01.  argv: mode (det|hogwild),
groups (NEXT-3 two-level ring, default 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2005_13789_b200 import ne  # noqa: E402
from paper_2005_13789_b200.engine import Engine  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    mode = sys.argv[1] if len(sys.argv) > 1 else "det"
    groups = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def all_gather(b: bytes):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    test = neg = None
    if mode == "hogwild":
        w = synth.CONFIGS["c1"]
        u, v = synth.rmat_edges(w.n, w.m, w.graph_seed)
        off, tgt, test = synth.split_edges(w.n, u, v, 0.1, synth.EVAL_SEED)
        neg = synth.negative_pairs(w.n, u, v, len(test), synth.EVAL_SEED + 1)
        epochs, kw = 5, dict(dim=128, walk_len=40, window=5, episodes=2, subparts=4)
    else:
        off, tgt = synth.rmat_graph(3000, 24000, 11)
        epochs, kw = 2, dict(dim=64, walk_len=12, window=3, episodes=2, subparts=3)
    kw["groups"] = groups
    n = len(off) - 1
    eng = Engine(deterministic=(mode == "det"), device=dev, rank=rank, world=world, nccl_id=None,
                 transport=ne.NE_TRANSPORT_IPC, **kw)
    eng.load_graph(off, tgt, all_gather=all_gather)
    a, b = eng.part
    exp = torch.full((b - a, kw["dim"]), float("nan")).pin_memory()  # rows streamed out on arrival home
    eng.export_vertex_on_train(exp)
    stats = [eng.train_epoch(ep, 0.025) for ep in range(epochs)]
    assert np.array_equal(exp.numpy(), eng.embeddings(0)), "exported vertex rows differ from ne_get_embeddings"
    if mode == "det":  # a reload of the same graph keeps the ring connected and restarts it
        eng.load_graph(off, tgt, all_gather=all_gather)
        stats = [eng.train_epoch(ep, 0.025) for ep in range(epochs)]
    V, Cm = eng.embeddings(0), eng.embeddings(1)
    assert np.array_equal(exp.numpy(), V), "exported vertex rows differ from ne_get_embeddings"
    parts = [None] * world
    dist.all_gather_object(parts, (a, b, V, Cm, stats))
    if rank == 0:
        cfg = oracle.Config(negatives=5, walks_per_node=1, parts=world, seed=42, **kw)
        Vr = oracle.init_vertex(n, kw["dim"], 42)
        Cr = np.zeros_like(Vr)
        ns = sum(oracle.train_epoch(cfg, off, tgt, Vr, Cr, ep, 0.025)[0] for ep in range(epochs))
        got = sum(st["samples"] for p in parts for st in p[4])
        assert got == ns, (got, ns)
        Vg = np.concatenate([p[2] for p in parts])
        Cg = np.concatenate([p[3] for p in parts])
        if mode == "det":
            dv, dc = float(np.abs(Vg - Vr).max()), float(np.abs(Cg - Cr).max())
            print(f"IPC det world={world} groups={groups} samples={ns} max|dV|={dv:.3e} max|dC|={dc:.3e}", flush=True)
            assert dv <= 1e-4 and dc <= 1e-4, (dv, dc)
        else:
            a_ref = oracle.auc(oracle.score_pairs(Vr, Cr, test), oracle.score_pairs(Vr, Cr, neg))
            a_gpu = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
            print(f"IPC hogwild world={world} AUC gpu {a_gpu:.4f} oracle {a_ref:.4f}", flush=True)
            assert abs(a_gpu - a_ref) <= 0.01, (a_gpu, a_ref)
    dist.barrier()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
