"""Oracle pins for O4 (walks), O5 (window pairs), O6 (canonical order and 2D
blocks) and O8 (negatives).  Expected values come from SPEC's worked examples,
closed forms, graph invariants (BFS reachability, stationary distribution) and
brute-force enumeration."""
from collections import Counter, deque

import numpy as np
import pytest

import synth
from conftest import golden_lines


# ---------------------------------------------------------------- O4 walks
def test_walk_chain_isolated(orc):
    off, tgt = synth.chain_graph(4)
    assert orc.random_walk(off, tgt, 42, 0, 0, 3).tolist() == [0, 1, 2, 3]
    assert orc.random_walk(off, tgt, 42, 0, 0, 10).tolist() == [0, 1, 2, 3]    # sink at 3
    off, tgt = synth.csr_from_directed(3, np.array([0]), np.array([1]))
    assert orc.random_walk(off, tgt, 42, 0, 2, 5).tolist() == [2]


def test_walk_star_uniform(orc):
    off, tgt = synth.star_graph(4)
    cnt = Counter()
    trials = 100_000
    for w in range(trials):
        p = orc.random_walk(off, tgt, 7, 0, w * 5, 1)   # omega = r*n + 0 (start 0)
        cnt[int(p[1])] += 1
    for leaf in range(1, 5):
        assert abs(cnt[leaf] / trials - 0.25) < 0.01


def test_walk_steps_are_edges_and_deterministic(orc):
    off, tgt = synth.rmat_graph(500, 3000, 11)
    edges = set()
    for u in range(500):
        for e in range(int(off[u]), int(off[u + 1])):
            edges.add((u, int(tgt[e])))
    for w in range(0, 1500, 7):
        p = orc.random_walk(off, tgt, 99, 3, w, 40)
        assert int(p[0]) == w % 500
        for a, b in zip(p[:-1], p[1:]):
            assert (int(a), int(b)) in edges
        if len(p) < 41:
            assert off[p[-1] + 1] == off[p[-1]]                                # only sinks stop
        assert np.array_equal(p, orc.random_walk(off, tgt, 99, 3, w, 40))
    a = orc.random_walk(off, tgt, 99, 3, 1, 40)
    b = orc.random_walk(off, tgt, 99, 4, 1, 40)
    assert not np.array_equal(a, b)   # the epoch enters the counter


def test_walk_stationary_distribution(orc):
    # connected, non-bipartite undirected graph: visit frequency -> deg / 2m
    u = np.array([0, 0, 1, 2, 3, 3, 4, 5, 5, 1])
    v = np.array([1, 2, 2, 3, 4, 5, 5, 0, 2, 4])
    off, tgt = synth.csr_from_undirected(6, u, v)
    deg = np.diff(off.astype(np.int64))
    steps = 300_000
    p = orc.random_walk(off, tgt, 5, 0, 0, steps)
    assert len(p) == steps + 1
    freq = np.bincount(p.astype(np.int64), minlength=6) / len(p)
    assert np.abs(freq - deg / deg.sum()).max() < 0.01


# ---------------------------------------------------------------- O5 pairs
def test_pair_counts_examples(orc):
    for row in golden_lines("augment_examples.txt"):
        if row.startswith("count"):
            lhs, rhs = row[len("count"):].split("->")
            walks, k, l = [int(x) for x in lhs.split()]
            assert walks * orc.pairs_per_walk(k, l) == int(rhs)
    for k in range(1, 9):
        for l in range(1, 9):
            lc = min(l, k)
            assert orc.pairs_per_walk(k, l) == k * lc - lc * (lc - 1) // 2


def test_pair_slot_order(orc):
    k, l = 5, 3
    got = [orc.pair_slot(k, l, s) for s in range(orc.pairs_per_walk(k, l))]
    exp = [(i, d) for i in range(k) for d in range(1, l + 1) if i + d <= k]
    assert got == exp


def _cfg(orc, **kw):
    base = dict(dim=8, negatives=2, walk_len=3, window=2, walks_per_node=1, episodes=1,
                subparts=1, parts=1, seed=42)
    base.update(kw)
    return orc.Config(**base)


def test_augment_worked_example(orc):
    # chain a->b->c->d, walk from a with k=3, l=2
    row = [r for r in golden_lines("augment_examples.txt") if r.startswith("path")][0]
    exp = sorted(tuple(int(x) for x in p.split(",")) for p in row.split("->")[1].split())
    off, tgt = synth.chain_graph(4)
    cfg = _cfg(orc, walk_len=3, window=2)
    pairs, boff = orc.build_episode(cfg, off, tgt, 0, 0)
    # walkers 1,2,3 start at b, c, d and add their own (shorter) pairs
    from_a = [tuple(map(int, p)) for p in pairs if True]
    walks = {0: [0, 1, 2, 3], 1: [1, 2, 3], 2: [2, 3], 3: [3]}
    expect_all = []
    for path in walks.values():
        for i in range(len(path)):
            for d in range(1, 3):
                if i + d < len(path):
                    expect_all.append((path[i], path[i + d]))
    assert sorted(from_a) == sorted(expect_all)
    assert sorted(p for p in expect_all[:5]) == exp


# ---------------------------------------------------------------- O6 order
def test_feistel_bits(orc):
    assert [orc.feistel_bits(N) for N in (1, 2, 3, 4, 5, 16, 17, 1 << 20, (1 << 20) + 1)] == \
           [2, 2, 2, 2, 3, 4, 5, 20, 21]


@pytest.mark.parametrize("N", list(range(1, 130)) + [255, 256, 257, 1000, 4097])
def test_feistel_is_bijection(orc, N):
    ys = [orc.feistel(x, N, 3, 1, 42) for x in range(N)]
    assert sorted(ys) == list(range(N))


def test_feistel_depends_on_episode_epoch_seed(orc):
    N = 1000
    base = [orc.feistel(x, N, 0, 0, 42) for x in range(N)]
    for args in [(1, 0, 42), (0, 1, 42), (0, 0, 43)]:
        assert [orc.feistel(x, N, *args) for x in range(N)] != base
    assert base != list(range(N))


def _bfs_within(off, tgt, src, limit):
    seen = {src: 0}
    q = deque([src])
    while q:
        u = q.popleft()
        if seen[u] == limit:
            continue
        for e in range(int(off[u]), int(off[u + 1])):
            v = int(tgt[e])
            if v not in seen:
                seen[v] = seen[u] + 1
                q.append(v)
    return seen


def test_episode_pool_counts_reachability_blocks(orc):
    n = 300
    off, tgt = synth.rmat_graph(n, 1500, 21)
    k, l = 10, 3
    cfg = _cfg(orc, walk_len=k, window=l, walks_per_node=2, parts=3, subparts=2)
    pairs, boff = orc.build_episode(cfg, off, tgt, 2, 0)
    # count = sum over walks of sum_delta (len - delta)
    expect = 0
    for w in range(2 * n):
        ln = len(orc.random_walk(off, tgt, 42, 2, w, k))
        expect += sum(max(0, ln - d) for d in range(1, l + 1))
    assert len(pairs) == expect
    # every sample reachable within min(l, k) hops
    for s in np.unique(pairs[:, 0])[:40]:
        reach = _bfs_within(off, tgt, int(s), min(l, k))
        for d in pairs[pairs[:, 0] == s][:, 1]:
            assert int(d) in reach
    # block membership: (vertex sub-part of src, context part of dst)
    P, ks = 3, 2
    pb = orc.partition_bounds(0, n, P).astype(np.int64)
    for B in range(P * ks * P):
        blk = pairs[int(boff[B]):int(boff[B + 1])]
        vs, cp = divmod(B, P)
        vp, t = divmod(vs, ks)
        sb = orc.partition_bounds(int(pb[vp]), int(pb[vp + 1]), ks).astype(np.int64)
        assert ((blk[:, 0] >= sb[t]) & (blk[:, 0] < sb[t + 1])).all()
        assert ((blk[:, 1] >= pb[cp]) & (blk[:, 1] < pb[cp + 1])).all()


def _generation_order(orc, off, tgt, cfg, epoch, episode):
    """The episode's pairs in generation order (O5): walkers ascending, window
    slots i-major / delta-minor, holes skipped -- from the pinned walk."""
    n = len(off) - 1
    u0, units = orc.episode_units(cfg, n, len(tgt), episode)
    out = []
    for w in range(u0, u0 + units):
        path = orc.random_walk(off, tgt, cfg.seed, epoch, w, cfg.walk_len)
        for i in range(cfg.walk_len):
            for d in range(1, cfg.window + 1):
                if i + d <= cfg.walk_len and i + d < len(path):
                    out.append((int(path[i]), int(path[i + d])))
    return out


def test_canonical_order_single_part(orc):
    # P = 1, one sub-part: pool[pi(x)] is the x-th generated pair, pi the
    # Feistel bijection over the episode's N pairs (O6)
    off, tgt = synth.rmat_graph(200, 1000, 5)
    cfg = _cfg(orc, walk_len=6, window=2)
    gen = _generation_order(orc, off, tgt, cfg, 4, 0)
    pool, _ = orc.build_episode(cfg, off, tgt, 4, 0)
    N = len(gen)
    assert len(pool) == N
    for x, pair in enumerate(gen):
        assert tuple(pool[orc.feistel(x, N, 0, 4, cfg.seed)]) == pair


def test_canonical_order_per_part(orc):
    # P = 2, k = 2: pairs of context part g, in generation order, get local
    # indices 0..N_g-1; inside every block the order is ascending pi_g(index)
    n = 200
    off, tgt = synth.rmat_graph(n, 1000, 5)
    cfg = _cfg(orc, walk_len=6, window=2, parts=2, subparts=2)
    gen = _generation_order(orc, off, tgt, cfg, 0, 0)
    pool, boff = orc.build_episode(cfg, off, tgt, 0, 0)
    pb = orc.partition_bounds(0, n, 2).astype(np.int64)
    part = [int(np.searchsorted(pb, d, side="right") - 1) for _, d in gen]
    Ng = [part.count(0), part.count(1)]
    nxt, keyed = [0, 0], []
    for (s_, d), g in zip(gen, part):
        vp = int(np.searchsorted(pb, s_, side="right") - 1)
        sb = orc.partition_bounds(int(pb[vp]), int(pb[vp + 1]), 2).astype(np.int64)
        t = int(np.searchsorted(sb, s_, side="right") - 1)
        B = (vp * 2 + t) * 2 + g
        keyed.append((B, orc.feistel(nxt[g], Ng[g], 0, 0, cfg.seed), (s_, d)))
        nxt[g] += 1
    keyed.sort()
    assert [k[2] for k in keyed] == [tuple(p) for p in pool.tolist()]
    assert [int(x) for x in boff] == [sum(1 for k in keyed if k[0] < B) for B in range(9)]


def test_episodes_partition_the_epoch(orc):
    n = 150
    off, tgt = synth.rmat_graph(n, 700, 8)
    whole, _ = orc.build_episode(_cfg(orc, walk_len=8, window=3), off, tgt, 1, 0)
    parts = [orc.build_episode(_cfg(orc, walk_len=8, window=3, episodes=4), off, tgt, 1, e)[0]
             for e in range(4)]
    assert sorted(map(tuple, whole.tolist())) == sorted(map(tuple, np.concatenate(parts).tolist()))


def test_line_mode_pool_is_edge_list(orc):
    n = 120
    off, tgt = synth.rmat_graph(n, 500, 9)
    pairs, _ = orc.build_episode(_cfg(orc, walk_len=0, window=0), off, tgt, 0, 0)
    edges = [(u, int(tgt[e])) for u in range(n) for e in range(int(off[u]), int(off[u + 1]))]
    assert sorted(map(tuple, pairs.tolist())) == sorted(edges)


# ---------------------------------------------------------------- O8 negatives
def test_negatives_follow_partition_alias(orc):
    n = 400
    off, tgt = synth.rmat_graph(n, 3000, 4)
    cfg = _cfg(orc, negatives=5, parts=2, subparts=1)
    thr, al = orc.build_alias_tables(cfg, off)
    pb = orc.partition_bounds(0, n, 2).astype(np.int64)
    deg = np.diff(off.astype(np.int64))
    for g in range(2):
        cb, cn = int(pb[g]), int(pb[g + 1] - pb[g])
        cnt = np.zeros(cn)
        draws = 0
        for pos in range(6000):
            negs = orc.negatives(cfg, thr, al, cb, cn, 0, 0, g, pos)
            assert ((negs >= cb) & (negs < cb + cn)).all()
            cnt[negs - cb] += 1
            draws += len(negs)
        w = np.array([orc.weight075(int(d)) for d in deg[cb:cb + cn]])
        p = w / w.sum()
        assert cnt[p == 0].sum() == 0
        # total-variation distance from deg^0.75 / Z is small at 30k draws
        assert 0.5 * np.abs(cnt / draws - p).sum() < 0.08
    a = orc.negatives(cfg, thr, al, 0, int(pb[1]), 0, 0, 0, 17)
    assert np.array_equal(a, orc.negatives(cfg, thr, al, 0, int(pb[1]), 0, 0, 0, 17))
    assert not np.array_equal(a, orc.negatives(cfg, thr, al, 0, int(pb[1]), 0, 1, 0, 17))
