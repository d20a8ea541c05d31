"""GPU parity for NEXT-4 bf16 row storage (DESIGN reading D16) against the
bf16 oracle (oracle.Config(storage=1)).

Init and the host round trip are exact (O9 value / input rounded to nearest
even).  Deterministic training: the kernel computes in fp32 (tree reduction,
fused multiply-adds), the oracle in double, and both round every stored row to
bf16.  A pre-rounding difference of ~1e-7 relative flips the rounding of an
element that lies within that distance of a rounding boundary, by one bf16 ulp
(2^-8 relative).  A row that differs by an ulp feeds its next update, which
can round one more ulp apart, so the divergence grows by at most ~1 ulp per
later store of the row.  On a perfect matching (one-step walks) a row is
stored ~1+K times, so the bar there is: >= 99 % of elements bit-identical and
every element within 2 + K ulp of the oracle's (ulp at the larger magnitude,
floor 2^-14 * 2^-7).  Measured: <= 2 ulp at K <= 3, 3-4 ulp at K = 5-7,
>= 99.67 % identical.  Over a
full epoch a flip feeds every later update of its row and bf16 SGD amplifies
it, so the full-epoch checks are loss, norm and link-prediction AUC.
Hogwild mode (bf16x4 vector reduction of each delta): AUC within 0.01 of the
bf16 oracle, as for fp32."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

BF16 = 1


def engine(**kw):
    from paper_2005_13789_b200.engine import Engine
    base = dict(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                subparts=4, deterministic=True, seed=42, device=0, storage=BF16)
    base.update(kw)
    return Engine(**base)


def ocfg(**kw):
    base = dict(dim=128, negatives=5, walk_len=40, window=5, walks_per_node=1, episodes=1,
                subparts=4, parts=1, seed=42, storage=BF16)
    base.update(kw)
    return oracle.Config(**base)


def ulp_bf16(x):
    m = np.maximum(np.abs(x), 2.0**-14)
    return 2.0 ** (np.floor(np.log2(m)) - 7)


def close_bf16(got, ref):
    assert (got.view(np.uint32) & 0xFFFF == 0).all()  # representable
    same = np.mean(got == ref)
    err = np.abs(got.astype(np.float64) - ref) / ulp_bf16(np.maximum(np.abs(got), np.abs(ref)))
    return same, float(err.max())


@pytest.mark.parametrize("d", [128, 96, 100, 256])
def test_bf16_init_exact(d):
    off, tgt = synth.workload_graph("c1")
    eng = engine(dim=d)
    eng.load_graph(off, tgt)
    assert np.array_equal(eng.embeddings(0), oracle.round_bf16(oracle.init_vertex(len(off) - 1, d, 42)))
    assert not eng.embeddings(1).any()
    eng.close()


def test_bf16_set_get_round_trip():
    off, tgt = synth.workload_graph("c1")
    n = len(off) - 1
    eng = engine(dim=64)
    eng.load_graph(off, tgt)
    rng = np.random.default_rng(3)
    for which in (0, 1):
        x = rng.normal(0, 0.3, (n, 64)).astype(np.float32)
        eng.set_embeddings(which, 0, x)
        assert np.array_equal(eng.embeddings(which), oracle.round_bf16(x))
    eng.close()


def _det_run(kw, graph=None, lr=0.025):
    off, tgt = graph if graph is not None else synth.workload_graph("c1")
    n = len(off) - 1
    cfg = ocfg(**{k: v for k, v in kw.items() if k != "staging"})  # staging: where rows live, not what
    eng = engine(**kw)
    eng.load_graph(off, tgt)
    V = oracle.round_bf16(oracle.init_vertex(n, cfg.dim, 42))
    Cm = np.zeros_like(V)
    st = eng.train_epoch(0, lr)
    ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, 0, lr)
    assert st["samples"] == ns
    assert abs(st["loss_sum"] - loss) <= 1e-3 * abs(loss)
    out = [(eng.embeddings(0), V), (eng.embeddings(1), Cm)]
    eng.close()
    return out


def _matching(n=20000):
    u = np.arange(0, n, 2, dtype=np.int64)
    return synth.csr_from_undirected(n, u, u + 1)


@pytest.mark.parametrize("kw", [
    dict(negatives=0),
    dict(negatives=1),
    dict(),                                            # K = 5
    dict(dim=96, subparts=3),                          # 8-lane groups
    dict(dim=256, negatives=3),                        # 32-lane groups, R = 2
    dict(dim=64, negatives=7),                         # runtime K
    dict(update_rule=1),                               # accumulated rule
])
def test_bf16_deterministic_matching(kw):
    """Perfect matching, one-step walks: every vertex row is trained by one
    sample and every context row by ~1+K (negatives are uniform at equal
    degrees), so rounding flips cannot cascade far and the element-wise bar of
    the module docstring applies; a wrong rounding mode or write-back misses it
    by far (truncation alone moves ~half of all elements)."""
    K = kw.get("negatives", 5)
    for got, ref in _det_run(dict(kw, walk_len=1, window=1), graph=_matching()):
        same, err = close_bf16(got, ref)
        assert same >= 0.99 and err <= 2.0 + K, (kw, same, err)


@pytest.mark.parametrize("kw", [dict(), dict(update_rule=1)])
def test_bf16_deterministic_epoch(kw):
    """A full C1 epoch (hub context rows are stored thousands of times): a flip
    is a 2^-8 step that feeds every later update of its row, and bf16 SGD
    amplifies it -- measured: 33 % of elements bit-identical, relative
    Frobenius difference 0.106 at equal loss.  Checked: samples, loss (1e-3),
    representability and the norm bound; quality parity is the AUC tests."""
    for got, ref in _det_run(kw):
        assert (got.view(np.uint32) & 0xFFFF == 0).all()
        rel = np.linalg.norm(got.astype(np.float64) - ref) / np.linalg.norm(ref)
        print("bf16 full-epoch relative Frobenius difference", kw, rel, np.mean(got == ref))
        assert rel <= 0.2, (kw, rel)


def test_bf16_deterministic_auc_matches_oracle():
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    kw = dict(dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1)
    cfg = ocfg(**kw)
    V = oracle.round_bf16(oracle.init_vertex(n, 32, 42))
    Cm = np.zeros_like(V)
    eng = engine(**kw)
    eng.load_graph(off, tgt)
    for ep in range(2):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
        eng.train_epoch(ep, 0.05)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    Vg, Cg = eng.embeddings(0), eng.embeddings(1)
    a = oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg))
    eng.close()
    assert a_ref > 0.9 and abs(a - a_ref) <= 0.01, (a_ref, a)


def test_bf16_hogwild_auc_matches_oracle():
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    kw = dict(dim=32, walk_len=20, window=3, walks_per_node=4, subparts=1)
    cfg = ocfg(**kw)
    V = oracle.round_bf16(oracle.init_vertex(n, 32, 42))
    Cm = np.zeros_like(V)
    for ep in range(2):
        oracle.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    a_ref = oracle.auc(oracle.score_pairs(V, Cm, test), oracle.score_pairs(V, Cm, neg))
    aucs = []
    for _ in range(3):
        eng = engine(deterministic=False, **kw)
        eng.load_graph(off, tgt)
        for ep in range(2):
            eng.train_epoch(ep, 0.05)
        Vg, Cg = eng.embeddings(0), eng.embeddings(1)
        assert (Vg.view(np.uint32) & 0xFFFF == 0).all()
        aucs.append(oracle.auc(oracle.score_pairs(Vg, Cg, test), oracle.score_pairs(Vg, Cg, neg)))
        eng.close()
    assert all(abs(a - a_ref) <= 0.01 for a in aucs), (a_ref, aucs)


@pytest.mark.parametrize("P", [2, 4])
def test_bf16_ring_emulation_matching(P):
    """P layout-only ranks on one device (pointer hand-over in place of the
    NCCL ring, which moves bf16 sub-parts): the element-wise bar against the
    oracle's P-part bf16 epoch on the perfect matching."""
    from paper_2005_13789_b200 import ne
    off, tgt = _matching()
    n = len(off) - 1
    kw = dict(walk_len=1, window=1)
    engs = [engine(rank=g, world=P, **kw) for g in range(P)]
    for e in engs:
        e.load_graph(off, tgt)
        e.random_walk(0, 0)
        e.build_samples(0, 0)
    st = ne.ne_train_samples_local_ring([e.ctx for e in engs], 0, 0, 0.025)
    cfg = ocfg(parts=P, **kw)
    V = oracle.round_bf16(oracle.init_vertex(n, 128, 42))
    Cm = np.zeros_like(V)
    ns, loss = oracle.train_epoch(cfg, off, tgt, V, Cm, 0, 0.025)
    assert st.samples == ns
    for e in engs:
        a, b = e.part
        for got, ref in ((e.embeddings(0), V[a:b]), (e.embeddings(1), Cm[a:b])):
            same, err = close_bf16(got, ref)
            assert same >= 0.99 and err <= 2.0 + 5, (P, same, err)
        e.close()


def test_bf16_host_staged_matching():
    """bf16 rows with the vertex matrix in pinned host memory (NEXT-2 staging
    moves bf16 sub-parts): the element-wise bar on the perfect matching, and
    the host round trip through the staged matrix."""
    from paper_2005_13789_b200 import ne
    for got, ref in _det_run(dict(walk_len=1, window=1, staging=ne.NE_STAGE_HOST), graph=_matching()):
        same, err = close_bf16(got, ref)
        assert same >= 0.99 and err <= 2.0 + 5, (same, err)
    off, tgt = _matching()
    eng = engine(dim=64, staging=ne.NE_STAGE_HOST)
    eng.load_graph(off, tgt)
    x = np.random.default_rng(5).normal(0, 0.3, (len(off) - 1, 64)).astype(np.float32)
    eng.set_embeddings(0, 0, x)
    assert np.array_equal(eng.embeddings(0), oracle.round_bf16(x))
    eng.close()
