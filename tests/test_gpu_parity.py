"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact for walks, pools and negatives (integer work,
shared Philox contract), max-abs 1e-4 for deterministic-mode embeddings after
one epoch (BASELINE.json north_star), AUC within 0.01 for the Hogwild
production mode."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north_star: deterministic-mode embeddings within max-abs 1e-4 (fp32)


def engine(**kw):
    from paper_2005_13789_b200.engine import Engine
    base = dict(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                subparts=4, deterministic=True, seed=42, device=0)
    base.update(kw)
    return Engine(**base)


def ocfg(**kw):
    base = dict(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                subparts=4, parts=1, seed=42)
    base.update(kw)
    return oracle.Config(**base)


@pytest.fixture(scope="module")
def c1():
    return synth.workload_graph("c1")


# ---------------------------------------------------------------- O9 init
def test_init_bit_exact(c1):
    off, tgt = c1
    n = len(off) - 1
    for d in (128, 96, 100):
        eng = engine(dim=d)
        eng.load_graph(off, tgt)
        assert np.array_equal(eng.embeddings(0), oracle.init_vertex(n, d, 42))
        assert not eng.embeddings(1).any()
        eng.close()


# ---------------------------------------------------------------- O4 walks
@pytest.mark.parametrize("epoch", [0, 5])
def test_walks_bit_exact_c1(c1, epoch):
    off, tgt = c1
    n = len(off) - 1
    eng = engine(walks_per_node=2, episodes=3)
    eng.load_graph(off, tgt)
    for e in range(3):
        walks = eng.random_walk(epoch, e, export=True)
        u0, units = oracle.episode_units(ocfg(walks_per_node=2, episodes=3), n, len(tgt), e)
        assert walks.shape == (units, 41)
        for w in range(units):
            ref = oracle.random_walk(off, tgt, 42, epoch, u0 + w, 40)
            assert np.array_equal(walks[w, :len(ref)], ref)
            assert (walks[w, len(ref):] == 0xFFFFFFFF).all()
    eng.close()


# ---------------------------------------------------------------- O5/O6 pools
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_pool_bit_exact_c1(c1, P):
    off, tgt = c1
    k = 4
    ref, boff = oracle.build_episode(ocfg(parts=P, subparts=k), off, tgt, 2, 0)
    for g in range(P):
        eng = engine(rank=g, world=P)
        eng.load_graph(off, tgt)
        eng.random_walk(2, 0)
        total = eng.build_samples(2, 0)
        got_total = 0
        for vs in range(P * k):
            B = vs * P + g
            blk = eng.export_samples(vs)
            assert np.array_equal(blk, ref[int(boff[B]):int(boff[B + 1])]), (P, g, vs)
            got_total += len(blk)
        assert got_total == total
        eng.close()


@pytest.mark.parametrize("sink", ["keyed", "direct"])
@pytest.mark.parametrize("kind", ["walk", "line"])
def test_pool_sinks_bit_exact(c1, sink, kind, monkeypatch):
    """Both pool paths (keyed + radix passes, the default; direct pi-indexed
    scatter, used when HBM is short) against the oracle: C1 at P = 1 and 4 (one
    radix pass, hundreds of 8192-position windows, a ragged last one), C1 with
    4 walks per node (N ~ 5.6 M > 2^22: two radix passes) and a small graph whose
    pool is a single partial window."""
    if sink == "direct":
        monkeypatch.setenv("NE_POOL_DIRECT", "1")
    else:
        monkeypatch.delenv("NE_POOL_DIRECT", raising=False)
    small = synth.csr_from_undirected(60, *synth.planted_partition_edges(60, 3, 4.0, 1.0, 3))
    kw = dict(walk_len=0, window=0) if kind == "line" else {}
    cases = [(c1, 1, 1), (c1, 4, 1), (small, 1, 1)] + ([(c1, 1, 4)] if kind == "walk" else [])
    for (off, tgt), P, wpn in cases:
        k = 3
        ref, boff = oracle.build_episode(ocfg(parts=P, subparts=k, walks_per_node=wpn, **kw), off, tgt, 4, 0)
        for g in range(P):
            eng = engine(rank=g, world=P, subparts=k, walks_per_node=wpn, **kw)
            eng.load_graph(off, tgt)
            if not kw:
                eng.random_walk(4, 0)
            total = eng.build_samples(4, 0)
            if P == 1:
                assert total == int(boff[-1])
            for vs in range(P * k):
                B = vs * P + g
                assert np.array_equal(eng.export_samples(vs), ref[int(boff[B]):int(boff[B + 1])]), (P, g, vs, wpn)
            eng.close()


@pytest.mark.parametrize("direct", ["0", "1"])
def test_pool_buffers_grow(direct, monkeypatch):
    """Pool buffers are sized by the first pool built (plus 1/8) and kept
    across same-shape reloads; a larger pool grows them.  R-MAT (84 550 pairs)
    -> uniform graph of the same n, nnz (114 000: growth) -> R-MAT again, two
    episodes each: every pool equals the oracle's."""
    monkeypatch.setenv("NE_POOL_DIRECT", direct)
    A = synth.rmat_graph(600, 3000, 21)
    B = synth.uniform_graph(600, 3000, 22)
    kw = dict(dim=32, episodes=2, subparts=2)
    cfg = ocfg(**kw)
    eng = engine(**kw)
    for off, tgt in (A, B, A):
        eng.load_graph(off, tgt)
        for e in (1, 0):
            ref, boff = oracle.build_episode(cfg, off, tgt, 6, e)
            eng.random_walk(6, e)
            assert eng.build_samples(6, e) == int(boff[-1])
            for vs in range(2):
                assert np.array_equal(eng.export_samples(vs), ref[int(boff[vs]):int(boff[vs + 1])]), (e, vs)
    eng.close()


@pytest.mark.parametrize("maxbits", ["3", "2", "1"])
def test_pool_many_radix_passes(c1, maxbits, monkeypatch):
    """The radix passes with a lowered bits-per-pass cap (C1's ~1.4 M-pair pool
    has 8 key bits above the window: 3 / 4 / 8 passes at P = 1, 2 / 3 / 6 at
    P = 4): the multi-pass region arithmetic that pools above 2^31 pairs use
    (3 passes at the default cap), bit-exact against the oracle."""
    monkeypatch.setenv("NE_RADIX_MAXBITS", maxbits)
    monkeypatch.delenv("NE_POOL_DIRECT", raising=False)
    off, tgt = c1
    for P in (1, 4):
        ref, boff = oracle.build_episode(ocfg(parts=P, subparts=3), off, tgt, 5, 0)
        for g in range(P):
            eng = engine(rank=g, world=P, subparts=3)
            eng.load_graph(off, tgt)
            eng.random_walk(5, 0)
            eng.build_samples(5, 0)
            for vs in range(P * 3):
                B = vs * P + g
                assert np.array_equal(eng.export_samples(vs), ref[int(boff[B]):int(boff[B + 1])]), (maxbits, P, g, vs)
            eng.close()


def test_pool_bit_exact_multi_episode_line(c1):
    off, tgt = c1
    for kw in (dict(episodes=3, walks_per_node=2, subparts=2), dict(walk_len=0, window=0, episodes=2)):
        cfg = ocfg(**kw)
        for e in range(cfg.episodes):
            ref, boff = oracle.build_episode(cfg, off, tgt, 1, e)
            eng = engine(**kw)
            eng.load_graph(off, tgt)
            if cfg.walk_len:
                eng.random_walk(1, e)
            eng.build_samples(1, e)
            for vs in range(cfg.subparts):
                assert np.array_equal(eng.export_samples(vs), ref[int(boff[vs]):int(boff[vs + 1])])
            eng.close()


# ---------------------------------------------------------------- O8 negatives
@pytest.mark.parametrize("P", [1, 4])
def test_negatives_bit_exact(c1, P):
    off, tgt = c1
    n = len(off) - 1
    cfg = ocfg(parts=P)
    thr, al = oracle.build_alias_tables(cfg, off)
    pb = oracle.partition_bounds(0, n, P).astype(np.int64)
    rng = np.random.default_rng(0)
    for g in range(P):
        eng = engine(rank=g, world=P)
        eng.load_graph(off, tgt)
        for vs in (0, P * 4 - 1):
            got = eng.export_negatives(7, 3, vs, 1000, 2000)
            for i in rng.integers(0, 2000, 300):
                ref = oracle.negatives(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 7, 3,
                                       vs * P + g, 1000 + int(i))
                assert np.array_equal(got[i], ref)
        eng.close()


# ---------------------------------------------------------------- O10/O11 training
def _det_epoch(off, tgt, epochs=1, lr=0.025, **kw):
    n = len(off) - 1
    cfg = ocfg(**{k: v for k, v in kw.items() if k not in ("deterministic", "conflict_permille", "writeback", "staging",
                                                           "stage_window")})
    eng = engine(**kw)
    eng.load_graph(off, tgt)
    V = oracle.init_vertex(n, cfg.dim, 42)
    Cm = np.zeros_like(V)
    for ep in range(epochs):
        st = eng.train_epoch(ep, lr)
        ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, ep, lr)
        assert st["samples"] == ns
        assert abs(st["loss_sum"] - loss) <= 1e-3 * abs(loss) + 1e-6
    dv = np.abs(eng.embeddings(0) - V).max()
    dc = np.abs(eng.embeddings(1) - Cm).max()
    eng.close()
    return dv, dc


def test_deterministic_epoch_c1():
    off, tgt = synth.workload_graph("c1")
    dv, dc = _det_epoch(off, tgt)
    assert dv <= TOL and dc <= TOL, (dv, dc)


@pytest.mark.parametrize("writeback", [0, 1])
def test_hogwild_code_path_single_warp_c1(writeback):
    """The production (Hogwild) kernel -- atomic-delta or store write-back --
    capped to one warp (conflict_permille=1) runs the block in canonical order,
    so it must match the oracle like the deterministic mode."""
    off, tgt = synth.workload_graph("c1")
    dv, dc = _det_epoch(off, tgt, deterministic=False, conflict_permille=1, writeback=writeback)
    assert dv <= TOL and dc <= TOL, (dv, dc)


@pytest.mark.parametrize("kw", [
    dict(dim=4, negatives=0, walk_len=5, window=2),
    dict(dim=96, negatives=8, walk_len=12, window=4, subparts=3, episodes=2),
    dict(dim=256, negatives=2, walk_len=8, window=8, walks_per_node=3),
    dict(dim=100, negatives=5, walk_len=0, window=0, episodes=2),
    dict(dim=96, negatives=5, walk_len=10, window=3),              # 8-lane groups (C4's d)
    dict(dim=80, negatives=5, walk_len=10, window=3, subparts=2),  # 8 lanes, ragged last float4
])
def test_deterministic_shapes(kw):
    off, tgt = synth.rmat_graph(700, 4000, 3)
    dv, dc = _det_epoch(off, tgt, epochs=2, **kw)
    assert dv <= TOL and dc <= TOL, (dv, dc)


def test_reuse_samples_and_repeat():
    off, tgt = synth.rmat_graph(300, 2000, 4)
    n = len(off) - 1
    eng = engine(dim=32)
    eng.load_graph(off, tgt)
    eng.train_epoch(0, 0.025)
    eng.train_epoch(1, 0.025, reuse=True)  # walk reuse: same pool, epoch-1 negatives
    cfg = ocfg(dim=32)
    V = oracle.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.025)
    # replay the epoch-0 pool with epoch-1 negatives
    pairs, boff = oracle.build_episode(cfg, off, tgt, 0, 0)
    thr, al = oracle.build_alias_tables(cfg, off)
    for t in range(4):
        for p in range(int(boff[t + 1] - boff[t])):
            s, d = pairs[int(boff[t]) + p]
            negs = oracle.negatives(cfg, thr, al, 0, n, 1, 0, t, p)
            oracle.train_sample(V, Cm, int(s), int(d), negs, 0.025)
    assert np.abs(eng.embeddings(0) - V).max() <= TOL
    assert np.abs(eng.embeddings(1) - Cm).max() <= TOL
    eng.close()


def test_hogwild_auc_matches_oracle():
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    kw = dict(dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1)
    cfg = ocfg(**kw)
    V = oracle.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    for ep in range(2):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    aucs = []
    for seed_run in range(3):
        eng = engine(deterministic=False, **kw)
        eng.load_graph(off, tgt)
        for ep in range(2):
            eng.train_epoch(ep, 0.05)
        Vg, Cg = eng.embeddings(0), eng.embeddings(1)
        aucs.append(oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg)))
        eng.close()
    assert all(abs(a - a_ref) <= 0.01 for a in aucs), (a_ref, aucs)


# ---------------------------------------------------------------- edges and errors
def test_empty_and_isolated_graphs():
    off = np.zeros(11, np.uint64)
    tgt = np.zeros(0, np.uint32)
    eng = engine(dim=8)
    eng.load_graph(off, tgt)
    walks = eng.random_walk(0, 0, export=True)
    assert (walks[:, 0] == np.arange(10)).all() and (walks[:, 1:] == 0xFFFFFFFF).all()
    assert eng.build_samples(0, 0) == 0
    st = eng.train_samples(0, 0, 0.025)
    assert st["samples"] == 0
    assert np.array_equal(eng.embeddings(0), oracle.init_vertex(10, 8, 42))
    eng.close()


def test_invalid_csr_rejected():
    from paper_2005_13789_b200 import ne
    eng = engine(dim=8)
    with pytest.raises(ne.NEError, match=r"NE_EINVAL: offsets\[2\]=1 < offsets\[1\]=3"):
        eng.load_graph(np.array([0, 3, 1, 4], np.uint64), np.array([1, 2, 0, 1], np.uint32))
    with pytest.raises(ne.NEError, match=r"NE_EINVAL: targets\[1\]=7 >= n=3"):
        eng.load_graph(np.array([0, 1, 2, 2], np.uint64), np.array([1, 7], np.uint32))
    with pytest.raises(ne.NEError, match=r"NE_EINVAL: offsets\[3\]=2 != nnz=3"):
        eng.load_graph(np.array([0, 1, 2, 2], np.uint64), np.array([1, 2, 0], np.uint32))
    with pytest.raises(ne.NEError, match="NE_ESTATE"):
        eng.train_epoch(0, 0.1)
    off, tgt = synth.chain_graph(5)
    eng.load_graph(off, tgt)
    with pytest.raises(ne.NEError, match="NE_ESTATE"):
        eng.build_samples(0, 0)  # no walks yet
    with pytest.raises(ne.NEError, match="NE_ERANGE"):
        eng.embeddings(0, rows=(0, 6))
    eng.close()


# ---------------------------------------------------------------- full size (C2)
def test_c2_full_size_sampled():
    off, tgt = synth.workload_graph("c2")
    n = len(off) - 1
    eng = engine(deterministic=False)
    eng.load_graph(off, tgt)
    walks = eng.random_walk(0, 0, export=True)
    rng = np.random.default_rng(1)
    for w in rng.integers(0, n, 3000):
        ref = oracle.random_walk(off, tgt, 42, 0, int(w), 40)
        assert np.array_equal(walks[w, :len(ref)], ref)
    lens = (walks != 0xFFFFFFFF).sum(1)
    expect = sum(np.maximum(lens - dl, 0).sum() for dl in range(1, 6))
    total = eng.build_samples(0, 0)
    assert total == expect
    cfg = ocfg()
    thr, al = oracle.build_alias_tables(cfg, off)
    for vs in range(4):
        blk = eng.export_samples(vs)
        sb = oracle.partition_bounds(0, n, 4).astype(np.int64)
        assert ((blk[:, 0] >= sb[vs]) & (blk[:, 0] < sb[vs + 1])).all()
        for p in rng.integers(0, len(blk), 200):
            got = eng.export_negatives(0, 0, vs, int(p), 1)[0]
            assert np.array_equal(got, oracle.negatives(cfg, thr, al, 0, n, 0, 0, vs, int(p)))
    st = eng.train_samples(0, 0, 0.025)
    assert st["samples"] == total and np.isfinite(st["loss_sum"])
    V = eng.embeddings(0)
    assert np.isfinite(V).all()
    eng.close()


def test_pool_keyed_equals_direct_c2(monkeypatch):
    """Full-size C2 pool (N ~ 10^8 > 2^22: two radix passes, ~13 000 windows):
    the keyed path equals the direct pi-indexed scatter block by block (both
    are pinned to the oracle on C1 by test_pool_sinks_bit_exact)."""
    off, tgt = synth.workload_graph("c2")
    pools = []
    for direct in ("0", "1"):
        monkeypatch.setenv("NE_POOL_DIRECT", direct)
        eng = engine(deterministic=False)
        eng.load_graph(off, tgt)
        eng.random_walk(3, 0)
        total = eng.build_samples(3, 0)
        assert total > (1 << 22)
        pools.append([eng.export_samples(vs) for vs in range(4)])
        eng.close()
    for a, b in zip(*pools):
        assert np.array_equal(a, b)


# ---------------------------------------------------------------- P-rank ring on one GPU
@pytest.mark.parametrize("P,G", [(2, 1), (4, 1), (8, 1), (4, 2), (8, 2), (8, 4)])
def test_deterministic_ring_emulation_c1(c1, P, G):
    """P layout-only ranks on one device, ring plan with pointer hand-over in
    place of ncclSend/Recv: embeddings within 1e-4 of the oracle's P-part epoch.
    G > 1: the NEXT-3 two-level plan (G groups of P/G ranks)."""
    from paper_2005_13789_b200 import ne
    off, tgt = c1
    n = len(off) - 1
    engs = [engine(rank=g, world=P, groups=G) for g in range(P)]
    total = 0
    for e in engs:
        e.load_graph(off, tgt)
        e.random_walk(0, 0)
        total += e.build_samples(0, 0)
    st = ne.ne_train_samples_local_ring([e.ctx for e in engs], 0, 0, 0.025)
    cfg = ocfg(parts=P, groups=G)
    V = oracle.init_vertex(n, 128, 42)
    Cm = np.zeros_like(V)
    ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.025)
    assert st.samples == ns == total
    assert abs(st.loss_sum - loss) <= 1e-3 * loss
    for e in engs:
        a, b = e.part
        assert np.abs(e.embeddings(0) - V[a:b]).max() <= TOL
        assert np.abs(e.embeddings(1) - Cm[a:b]).max() <= TOL
        e.close()


@pytest.mark.parametrize("P,w", [(2, 2), (4, 2), (4, 1), (2, 4)])
def test_staged_ring_emulation_c1(c1, P, w):
    """NEXT-2 with the ring (reading D18): every rank's vertex part in pinned
    host memory, its sub-parts going around the ring in windows of w slots
    (H2D of the window, P rounds with hand-over, D2H) -- P layout-only ranks on
    one device: within 1e-4 of the oracle's windowed plan."""
    from paper_2005_13789_b200 import ne
    off, tgt = c1
    n = len(off) - 1
    engs = [engine(rank=g, world=P, staging=1, stage_window=w) for g in range(P)]
    for e in engs:
        e.load_graph(off, tgt)
        e.random_walk(0, 0)
        e.build_samples(0, 0)
    st = ne.ne_train_samples_local_ring([e.ctx for e in engs], 0, 0, 0.025)
    cfg = ocfg(parts=P, window_slots=w)
    V = oracle.init_vertex(n, 128, 42)
    Cm = np.zeros_like(V)
    ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.025)
    assert st.samples == ns
    for e in engs:
        a, b = e.part
        assert np.abs(e.embeddings(0) - V[a:b]).max() <= TOL
        assert np.abs(e.embeddings(1) - Cm[a:b]).max() <= TOL
        e.close()


def test_reload_same_shape_graph_reuses_buffers():
    """ne_load_graph of a second graph with the same n and nnz reuses every
    device buffer; the result must be that of a fresh context."""
    offA, tgtA = synth.rmat_graph(600, 3000, 21)
    offB, tgtB = synth.uniform_graph(600, 3000, 22)
    assert len(tgtA) == len(tgtB)
    eng = engine(dim=32)
    eng.load_graph(offA, tgtA)
    eng.train_epoch(0, 0.025)
    eng.load_graph(offB, tgtB)
    assert np.array_equal(eng.embeddings(0), oracle.init_vertex(600, 32, 42))
    assert not eng.embeddings(1).any()
    eng.train_epoch(0, 0.025)
    cfg = ocfg(dim=32)
    V = oracle.init_vertex(600, 32, 42)
    Cm = np.zeros_like(V)
    oracle.train_epoch(cfg, offB, tgtB, V, Cm, 0, 0.025)
    assert np.abs(eng.embeddings(0) - V).max() <= TOL
    assert np.abs(eng.embeddings(1) - Cm).max() <= TOL
    eng.close()


# ---------------------------------------------------------------- NEXT-1 node2vec
@pytest.mark.parametrize("pq", [(0.5, 2.0), (4.0, 0.25), (1.0, 1.0)])
def test_node2vec_walks_and_pool_bit_exact(c1, pq):
    p, q = pq
    off, tgt = c1
    n = len(off) - 1
    eng = engine(p=p, q=q, walks_per_node=2, episodes=2, subparts=2)
    eng.load_graph(off, tgt)
    walks = eng.random_walk(3, 1, export=True)
    u0, units = oracle.episode_units(ocfg(walks_per_node=2, episodes=2), n, len(tgt), 1)
    for w in range(0, units, 3):
        ref = oracle.node2vec_walk(off, tgt, 42, 3, u0 + w, 40, p, q)
        assert np.array_equal(walks[w, :len(ref)], ref)
        assert (walks[w, len(ref):] == 0xFFFFFFFF).all()
    eng.build_samples(3, 1)
    ref, boff = oracle.build_episode(ocfg(p=p, q=q, walks_per_node=2, episodes=2, subparts=2), off, tgt, 3, 1)
    for vs in range(2):
        assert np.array_equal(eng.export_samples(vs), ref[int(boff[vs]):int(boff[vs + 1])])
    eng.close()


def test_node2vec_deterministic_epoch():
    off, tgt = synth.rmat_graph(900, 6000, 35)
    dv, dc = _det_epoch(off, tgt, epochs=1, dim=64, walk_len=20, window=4, p=0.25, q=4.0)
    assert dv <= TOL and dc <= TOL, (dv, dc)


def test_node2vec_requires_sorted_rows():
    from paper_2005_13789_b200 import ne
    off = np.array([0, 3, 4, 5, 6], np.uint64)
    tgt = np.array([3, 1, 2, 0, 0, 0], np.uint32)   # row 0 = [3, 1, 2] not sorted
    eng = engine(dim=8, p=0.5, q=2.0, walk_len=5, window=2)
    with pytest.raises(ne.NEError, match=r"NE_EINVAL: targets\[1\]=1 < targets\[0\]=3"):
        eng.load_graph(off, tgt)
    eng.close()
    eng = engine(dim=8, walk_len=5, window=2)      # first order: order does not matter
    eng.load_graph(off, tgt)
    eng.close()


@pytest.mark.parametrize("staged", ["0", "1"])
def test_hogwild_auc_gate_c1(staged, monkeypatch):
    """SURVEY 8(c) gate: production (Hogwild) AUC within 0.01 of the oracle on
    C1 with 10% held-out edges after 5 epochs (several production runs); also
    for the shared-memory-staged kernel (NE_SGNS_STAGED=1)."""
    monkeypatch.setenv("NE_SGNS_STAGED", staged)
    w = synth.CONFIGS["c1"]
    u, v = synth.rmat_edges(w.n, w.m, w.graph_seed)
    off, tgt, test = synth.split_edges(w.n, u, v, 0.1, synth.EVAL_SEED)
    neg = synth.negative_pairs(w.n, u, v, len(test), synth.EVAL_SEED + 1)
    cfg = ocfg()
    V = oracle.init_vertex(w.n, 128, 42)
    Cm = np.zeros_like(V)
    tables = oracle.build_alias_tables(cfg, off)
    for ep in range(5):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.025, tables=tables)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    aucs = []
    for run in range(3):
        eng = engine(deterministic=False)
        eng.load_graph(off, tgt)
        for ep in range(5):
            eng.train_epoch(ep, 0.025)
        Vg, Cg = eng.embeddings(0), eng.embeddings(1)
        aucs.append(oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg)))
        eng.close()
    assert all(abs(a - a_ref) <= 0.01 for a in aucs), (a_ref, aucs)


@pytest.mark.parametrize("P", [1, 4])
def test_pool_schedule_check(c1, P):
    """ne_check_pool: every pooled sample lies in its 2D block."""
    from paper_2005_13789_b200 import ne
    off, tgt = c1
    for g in range(P):
        eng = engine(rank=g, world=P, deterministic=False)
        eng.load_graph(off, tgt)
        eng.random_walk(0, 0)
        eng.build_samples(0, 0)
        ne.ne_check_pool(eng.ctx)
        eng.close()
    eng = engine(deterministic=False)
    eng.load_graph(off, tgt)
    st = ne.ne_train_epoch(eng.ctx, 0, 0.025, ne.NE_CHECK_BLOCKS)
    assert st.samples > 0
    eng.close()


# ---------------------------------------------------------------- NEXT-4 accumulated update
def test_accumulated_rule_deterministic_epoch_c1():
    off, tgt = synth.workload_graph("c1")
    dv, dc = _det_epoch(off, tgt, update_rule=1)
    assert dv <= TOL and dc <= TOL, (dv, dc)


def test_accumulated_rule_hogwild_auc():
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    kw = dict(dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1, update_rule=1)
    cfg = ocfg(**kw)
    V = oracle.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    for ep in range(2):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    eng = engine(deterministic=False, **kw)
    eng.load_graph(off, tgt)
    for ep in range(2):
        eng.train_epoch(ep, 0.05)
    Vg, Cg = eng.embeddings(0), eng.embeddings(1)
    a = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
    eng.close()
    assert abs(a - a_ref) <= 0.01, (a_ref, a)


# ---------------------------------------------------------------- NEXT-2 host staging
@pytest.mark.parametrize("subparts", [2, 3, 7])
def test_host_staged_vertex_matrix_matches_oracle(subparts):
    """NE_STAGE_HOST: the vertex matrix lives in pinned host memory and streams
    through 3 device slots (P:142 stages 2, 5); results equal the in-HBM path.
    k = 2, 3, 7 cover the next-episode prefetch of sub-part 0 with k < 3,
    k = 3 and a slot rotation that moves every episode (7 % 3 = 1)."""
    off, tgt = synth.rmat_graph(3000, 20000, 41)
    dv, dc = _det_epoch(off, tgt, epochs=2, dim=64, walk_len=12, window=3, subparts=subparts,
                        episodes=2, staging=1)
    assert dv <= TOL and dc <= TOL, (dv, dc)


@pytest.mark.parametrize("subparts,episodes", [(1, 1), (4, 2), (7, 3)])
def test_export_vertex_on_train(subparts, episodes):
    """ne_export_vertex_on_train: every train_epoch copies each vertex sub-part
    out as soon as its block of the last episode has trained; on return the
    host rows equal ne_get_embeddings(NE_VERTEX), across reloads; None stops it."""
    import torch
    off, tgt = synth.rmat_graph(3000, 20000, 44)
    eng = engine(dim=64, walk_len=10, window=3, subparts=subparts, episodes=episodes, deterministic=False)
    eng.load_graph(off, tgt)
    out = torch.full((3000, 64), float("nan"), dtype=torch.float32).pin_memory()
    eng.export_vertex_on_train(out)
    for ep in range(2):
        eng.train_epoch(ep, 0.025)
        assert np.array_equal(out.numpy(), eng.embeddings(0))
    eng.load_graph(off, tgt)  # the registration survives a reload
    eng.train_epoch(0, 0.025)
    assert np.array_equal(out.numpy(), eng.embeddings(0))
    eng.export_vertex_on_train(None)
    before = out.numpy().copy()
    eng.train_epoch(1, 0.025)
    assert np.array_equal(out.numpy(), before)
    eng.close()


def test_export_vertex_on_train_rejects():
    from paper_2005_13789_b200 import ne
    off, tgt = synth.rmat_graph(3000, 20000, 44)
    eng = engine(dim=64, walk_len=10, window=3)
    eng.load_graph(off, tgt)
    with pytest.raises(ne.NEError, match="NE_ERANGE"):
        eng.export_vertex_on_train(np.zeros((2999, 64), np.float32))
    eng.close()
    for kw, msg in ((dict(storage=ne.NE_STORE_BF16), "fp32 rows"), (dict(staging=ne.NE_STAGE_HOST), "device staging"),
                    (dict(rank=1, world=2), "layout-only")):
        eng = engine(dim=64, walk_len=10, window=3, **kw)
        with pytest.raises(ne.NEError, match=msg):
            eng.export_vertex_on_train(np.zeros((3000, 64), np.float32))
        eng.close()


def test_host_staged_write_drops_prefetch():
    """A host write between epochs lands after the next episode's sub-part 0
    was prefetched: the write must win (the prefetch is dropped), so the run
    still equals the oracle fed the same write."""
    off, tgt = synth.rmat_graph(3000, 20000, 43)
    kw = dict(dim=64, walk_len=10, window=3, subparts=7, episodes=2)
    cfg = ocfg(**kw)
    eng = engine(staging=1, **kw)
    eng.load_graph(off, tgt)
    V = oracle.init_vertex(3000, 64, 42)
    Cm = np.zeros_like(V)
    mark = np.random.default_rng(3).normal(0, 0.1, (40, 64)).astype(np.float32)
    for ep in range(2):
        eng.train_epoch(ep, 0.025)
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.025)
        eng.set_embeddings(0, 10, mark)   # rows of sub-part 0
        V[10:50] = mark
    assert np.abs(eng.embeddings(0) - V).max() <= TOL
    assert np.abs(eng.embeddings(1) - Cm).max() <= TOL
    eng.close()


def test_host_staged_set_get_and_hogwild():
    off, tgt = synth.rmat_graph(3000, 20000, 42)
    eng = engine(dim=32, walk_len=10, window=2, subparts=8, staging=1, deterministic=False)
    eng.load_graph(off, tgt)
    V = eng.embeddings(0)
    assert np.array_equal(V, oracle.init_vertex(3000, 32, 42))
    mark = np.full((5, 32), 0.25, np.float32)
    eng.set_embeddings(0, 100, mark)
    assert np.array_equal(eng.embeddings(0, rows=(100, 105)), mark)
    st = eng.train_epoch(0, 0.025)
    assert st["samples"] > 0 and np.isfinite(st["loss_sum"])
    V2 = eng.embeddings(0)
    assert np.isfinite(V2).all() and not np.array_equal(V2, V)
    eng.close()


# ---------------------------------------------------------------- production grid, position by position
def _matching(n):
    u = np.arange(0, n, 2, dtype=np.int64)
    return synth.csr_from_undirected(n, u, u + 1)


@pytest.mark.parametrize("dim,vsub,staged", [(128, 1, "0"), (96, 2, "0"), (128, 3, "1")])
def test_capture_ids_full_grid_c2(dim, vsub, staged, monkeypatch):
    """The production kernel at its full grid on C2 (d = 128: 16-lane groups,
    2 samples per warp; d = 96: 8-lane groups, 4 samples per warp) records the
    (src, dst, negatives) every group trained; every position must equal the
    pool and the oracle's negatives -- the lane -> sample -> negative routing
    of all S groups of a warp, checked at every position of the block."""
    monkeypatch.setenv("NE_SGNS_STAGED", staged)  # "1": the shared-memory-staged kernel
    off, tgt = synth.workload_graph("c2")
    n = len(off) - 1
    eng = engine(dim=dim, deterministic=False)
    eng.load_graph(off, tgt)
    eng.random_walk(0, 0)
    eng.build_samples(0, 0)
    pool = eng.export_samples(vsub)
    cap = eng.capture_block(0, 0, vsub, 0.025)
    assert cap.shape == (len(pool), 7) and len(pool) > 10_000_000
    assert np.array_equal(cap[:, :2], pool)
    cfg = ocfg(dim=dim)
    thr, al = oracle.build_alias_tables(cfg, off)
    ref = oracle.negatives_range(cfg, thr, al, 0, n, 0, 0, vsub, 0, len(pool))
    bad = np.flatnonzero((cap[:, 2:] != ref).any(1))
    assert len(bad) == 0, (len(bad), bad[:5], cap[bad[:3]], ref[bad[:3]])
    assert np.isfinite(eng.embeddings(0)).all()
    eng.close()


def test_capture_ids_layout_ranks_c1():
    """Capture at P = 4 (layout-only ranks): block ids vsub * P + rank in the
    negative counter, context-part alias tables."""
    off, tgt = synth.workload_graph("c1")
    n = len(off) - 1
    P = 4
    cfg = ocfg(parts=P)
    thr, al = oracle.build_alias_tables(cfg, off)
    pb = oracle.partition_bounds(0, n, P).astype(np.int64)
    for g in (0, 3):
        eng = engine(rank=g, world=P, deterministic=False)
        eng.load_graph(off, tgt)
        eng.random_walk(1, 0)
        eng.build_samples(1, 0)
        vs = g * 4 + 1
        pool = eng.export_samples(vs)
        cap = eng.capture_block(1, 0, vs, 0.025)
        assert np.array_equal(cap[:, :2], pool)
        ref = oracle.negatives_range(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 1, 0, vs * P + g, 0, len(pool))
        assert np.array_equal(cap[:, 2:], ref)
        eng.close()


@pytest.mark.parametrize("dim,staged", [(64, "0"), (128, "0"), (256, "0"), (128, "1")])
def test_hogwild_full_grid_conflict_free_elementwise(dim, staged, monkeypatch):
    """A perfect matching with walk_len = window = 1 and K = 0: every vertex row
    and every context row is touched by exactly one sample, so the production
    (Hogwild, atomic-delta) kernel at its full grid has no conflicts and must
    equal the oracle element by element (fp32 arithmetic vs the fp64 oracle)."""
    monkeypatch.setenv("NE_SGNS_STAGED", staged)
    n = 1 << 21
    off, tgt = _matching(n)
    kw = dict(dim=dim, negatives=0, walk_len=1, window=1)
    eng = engine(deterministic=False, **kw)
    eng.load_graph(off, tgt)
    st = eng.train_epoch(0, 0.025)
    assert st["samples"] == n
    V = oracle.init_vertex(n, dim, 42)
    Cm = np.zeros_like(V)
    ns, loss = oracle.train_epoch(ocfg(**kw), off, tgt, V, Cm, 0, 0.025)
    assert ns == n and abs(st["loss_sum"] - loss) <= 1e-5 * loss
    dv = np.abs(eng.embeddings(0) - V).max()
    dc = np.abs(eng.embeddings(1) - Cm).max()
    eng.close()
    assert dv <= 1e-6 and dc <= 1e-6, (dv, dc)


@pytest.mark.parametrize("deterministic", [True, False])
def test_sigmoid_clamp_in_kernel(deterministic):
    """The kernel's +-30 clamp (reading D11; tests/golden/sigma_clamp.txt): with
    lr = 0 the rows stay put and the loss of a positive sample with v.c = -40
    is log(1 + e^30) = 30 (no clamp: 40; a +-6 clamp: 6.0025), with v.c = -25
    it is 25."""
    from conftest import golden_kv
    g = golden_kv("sigma_clamp.txt")
    n, d = 4096, 8
    off, tgt = _matching(n)
    for dot, key in ((-40.0, "loss_pos_at_minus_40"), (-25.0, "loss_pos_at_minus_25")):
        eng = engine(dim=d, negatives=0, walk_len=1, window=1, deterministic=deterministic, subparts=1)
        eng.load_graph(off, tgt)
        eng.set_embeddings(0, 0, np.full((n, d), dot / d / -2.0, np.float32))
        eng.set_embeddings(1, 0, np.full((n, d), -2.0, np.float32))
        st = eng.train_epoch(0, 0.0)
        eng.close()
        assert st["samples"] == n
        assert abs(st["loss_sum"] / n - float(g[key])) <= 1e-4, (dot, st["loss_sum"] / n)


def test_c2_walks_and_pools_match_oracle_hashes():
    """C2 at full size (SURVEY 8(c) gate "walks and samples bit-exact on C2"):
    every walk and every 2D block of the pool at P = 1 and at P = 4
    (layout-only ranks), against SHA-256 hashes the oracle wrote
    (tests/golden/c2_hashes.txt, tools/make_golden_c2.py -- oracle only)."""
    import hashlib
    from conftest import golden_lines
    want_walk, want_blocks = None, {}
    for ln in golden_lines("c2_hashes.txt"):
        f = ln.split()
        if f[0] == "walks":
            want_walk = (int(f[1]), f[2])
        else:
            want_blocks[(int(f[1]), int(f[2]), int(f[3]))] = (int(f[4]), f[5])
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    off, tgt = synth.workload_graph("c2")
    n = len(off) - 1
    eng = engine(deterministic=False)
    eng.load_graph(off, tgt)
    walks = eng.random_walk(0, 0, export=True)
    assert (len(walks), sha(walks)) == want_walk
    del walks
    eng.close()
    for P in (1, 4):
        for g in range(P):
            eng = engine(deterministic=False, rank=g, world=P)
            eng.load_graph(off, tgt)
            eng.random_walk(3, 0)
            eng.build_samples(3, 0)
            for vs in range(P * 4):
                blk = eng.export_samples(vs)
                assert (len(blk), sha(blk)) == want_blocks[(P, g, vs)], (P, g, vs)
            eng.close()
