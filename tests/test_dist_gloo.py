"""Multi-process (world size 2, 3 and 4 with two groups, gloo, CPU) check of
the ring's host logic: every rank follows the library's schedule
(ne_plan_vsub2, ne_ring_peers, ne_partition_bounds from libne_b200.so, no GPU
needed), trains its block with the oracle's single-sample update, and ships
the trained vertex sub-part to the library's ring destination while receiving
the next from its ring source (torch.distributed send/recv) -- g+1 / g-1 on
one ring, the group ring or the next group with NEXT-3 groups.
The gathered result must be bit-identical to the oracle's sequential replay of
the P-part plan (P:89 orthogonality, S:383 sequential equivalence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, groups, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_2005_13789_b200 import ne

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, d, k = 260, 8, 2
        off, tgt = synth.rmat_graph(n, 1500, 13)
        cfg = oracle.Config(dim=d, negatives=3, walk_len=6, window=2, walks_per_node=1, episodes=2,
                            subparts=k, parts=world, seed=42, groups=groups)
        # NCCL-id bootstrap path of bench.py / the harness, over gloo
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        pb = ne.ne_partition_bounds(n, world).astype(np.int64)
        sb = np.concatenate([ne.ne_partition_bounds(int(pb[p + 1] - pb[p]), k).astype(np.int64)[:-1] + pb[p]
                             for p in range(world)] + [np.array([n])])
        V0 = oracle.init_vertex(n, d, 42)
        # my state: context part g (full-size scratch matrix, only my rows used)
        Cm = np.zeros((n, d), np.float32)
        slots = {t: (rank * k + t, V0[sb[rank * k + t]:sb[rank * k + t + 1]].copy()) for t in range(k)}
        thr, al = oracle.build_alias_tables(cfg, off)
        cb, cn = int(pb[rank]), int(pb[rank + 1] - pb[rank])
        for e in range(2):
            pairs, boff = oracle.build_episode(cfg, off, tgt, 0, e)
            for r in range(world):
                for t in range(k):
                    vs = ne.ne_plan_vsub2(world, groups, k, r, t, rank)
                    have, rows = slots[t]
                    assert have == vs, (rank, r, t, have, vs)
                    Vfull = np.zeros((n, d), np.float32)
                    Vfull[sb[vs]:sb[vs + 1]] = rows
                    B = vs * world + rank
                    for p in range(int(boff[B + 1] - boff[B])):
                        s, dd = pairs[int(boff[B]) + p]
                        negs = oracle.negatives(cfg, thr, al, cb, cn, 0, e, B, p)
                        oracle.train_sample(Vfull, Cm, int(s), int(dd), negs, 0.05)
                    rows = Vfull[sb[vs]:sb[vs + 1]].copy()
                    # ring: send to the library's destination, receive from its source
                    nxt = ne.ne_plan_vsub2(world, groups, k, r + 1, t, rank)
                    dest, src = ne.ne_ring_peers(world, groups, r, rank)
                    out = torch.from_numpy(rows)
                    inc = torch.zeros((int(sb[nxt + 1] - sb[nxt]), d), dtype=torch.float32)
                    reqs = [dist.isend(out, dest), dist.irecv(inc, src)]
                    for rq in reqs:
                        rq.wait()
                    slots[t] = (nxt, inc.numpy().copy())
        mine = {t: slots[t] for t in range(k)}
        q.put((rank, {t: (v[0], v[1]) for t, v in mine.items()}, Cm[cb:cb + cn].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,groups", [(2, 1), (3, 1), (4, 2)])
def test_ring_host_logic_matches_oracle(world, groups, orc):
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, groups, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, d, k = 260, 8, 2
    off, tgt = synth.rmat_graph(n, 1500, 13)
    cfg = orc.Config(dim=d, negatives=3, walk_len=6, window=2, walks_per_node=1, episodes=2,
                     subparts=k, parts=world, seed=42, groups=groups)
    V = orc.init_vertex(n, d, 42)
    Cm = np.zeros_like(V)
    orc.train_epoch(cfg, off, tgt, V, Cm, 0, 0.05)
    from paper_2005_13789_b200 import ne
    pb = ne.ne_partition_bounds(n, world).astype(np.int64)
    for rank, slots, cpart in results:
        assert np.array_equal(cpart, Cm[pb[rank]:pb[rank + 1]])
        sb = ne.ne_partition_bounds(int(pb[rank + 1] - pb[rank]), k).astype(np.int64) + pb[rank]
        for t, (vs, rows) in slots.items():
            assert vs == rank * k + t          # every sub-part is home after P rounds
            assert np.array_equal(rows, V[sb[t]:sb[t + 1]])
