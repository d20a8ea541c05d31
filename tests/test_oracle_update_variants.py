"""Oracle pins for NEXT-4, the accumulated-gradient update (word2vec /
GraphVite style): the vertex gradient of all 1+K pairs is taken at the
pre-sample vertex row and applied once.  Pins: finite differences of the
per-sample negative-sampling loss, one-exact-SGD-step equivalence, reduction to
the sequential rule for K = 0, in-place handling of repeated ids, learning."""
import numpy as np

import synth


def test_total_gradient_matches_finite_differences(orc):
    rng = np.random.default_rng(5)

    def total_loss(v, cs, labels):
        return orc.sgns_total_grad(v, cs, labels)[2]

    for _ in range(60):
        d = int(rng.integers(1, 17))
        m = int(rng.integers(1, 7))
        v = rng.normal(0, 0.6, d)
        cs = [rng.normal(0, 0.6, d) for _ in range(m)]
        labels = [1] + [0] * (m - 1)
        gv, gcs, _ = orc.sgns_total_grad(v, cs, labels)
        h = 1e-5
        fv = np.zeros(d)
        for i in range(d):
            e = np.zeros(d)
            e[i] = h
            fv[i] = (total_loss(v + e, cs, labels) - total_loss(v - e, cs, labels)) / (2 * h)
        assert np.linalg.norm(gv - fv) <= 1e-4 * max(np.linalg.norm(fv), 1e-12)
        for j in range(m):
            fc = np.zeros(d)
            for i in range(d):
                e = np.zeros(d)
                e[i] = h
                cp = [c.copy() for c in cs]
                cm = [c.copy() for c in cs]
                cp[j] += e
                cm[j] -= e
                fc[i] = (total_loss(v, cp, labels) - total_loss(v, cm, labels)) / (2 * h)
            assert np.linalg.norm(gcs[j] - fc) <= 1e-4 * max(np.linalg.norm(fc), 1e-12)


def test_accumulated_sample_is_one_sgd_step(orc):
    rng = np.random.default_rng(6)
    d, K, lr = 12, 5, 0.05
    V = rng.normal(0, 0.3, (8, d)).astype(np.float32)
    Cm = rng.normal(0, 0.3, (8, d)).astype(np.float32)
    negs = np.array([2, 3, 4, 5, 6], np.uint32)
    V1, C1 = V.copy(), Cm.copy()
    orc.train_sample_accumulated(V1, C1, 0, 1, negs, lr)
    ids = [1, 2, 3, 4, 5, 6]
    gv, gcs, _ = orc.sgns_total_grad(V[0].astype(np.float64), [Cm[i].astype(np.float64) for i in ids],
                                     [1, 0, 0, 0, 0, 0])
    assert np.allclose(V1[0], V[0] - lr * gv, atol=1e-6, rtol=0)
    for i, g in zip(ids, gcs):
        assert np.allclose(C1[i], Cm[i] - lr * g, atol=1e-6, rtol=0)
    assert np.array_equal(V1[1:], V[1:]) and np.array_equal(C1[[0, 7]], Cm[[0, 7]])


def test_single_pair_reduces_to_sequential(orc):
    rng = np.random.default_rng(7)
    V = rng.normal(0, 0.3, (3, 9)).astype(np.float32)
    Cm = rng.normal(0, 0.3, (3, 9)).astype(np.float32)
    V1, C1, V2, C2 = V.copy(), Cm.copy(), V.copy(), Cm.copy()
    l1 = orc.train_sample_accumulated(V1, C1, 0, 2, np.zeros(0, np.uint32), 0.1)
    l2 = orc.train_sample(V2, C2, 0, 2, np.zeros(0, np.uint32), 0.1)
    assert np.array_equal(V1, V2) and np.array_equal(C1, C2) and l1 == l2


def test_repeated_context_sees_earlier_update(orc):
    rng = np.random.default_rng(8)
    d = 6
    V = rng.normal(0, 0.4, (4, d)).astype(np.float32)
    Cm = rng.normal(0, 0.4, (4, d)).astype(np.float32)
    negs = np.array([2, 2, 1], np.uint32)      # 2 twice, and the positive id 1 again
    V1, C1 = V.copy(), Cm.copy()
    orc.train_sample_accumulated(V1, C1, 0, 1, negs, 0.1)
    # word2vec order: context rows updated in place with v0, v updated once
    v0 = V[0].astype(np.float64)
    c = Cm.astype(np.float64)
    e = np.zeros(d)
    for cid, y in [(1, 1), (2, 0), (2, 0), (1, 0)]:
        g = orc.sigmoid(float(v0 @ c[cid])) - y
        e += g * c[cid]
        c[cid] = (c[cid] - 0.1 * g * v0).astype(np.float32)
    assert np.allclose(C1, c.astype(np.float32), atol=2e-7, rtol=0)
    assert np.allclose(V1[0], (v0 - 0.1 * e).astype(np.float32), atol=2e-7, rtol=0)


def test_accumulated_epoch_learns(orc):
    n = 2000
    u, v = synth.planted_partition_edges(n, 20, 12.0, 1.0, 17)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    cfg = orc.Config(dim=32, negatives=5, walk_len=20, window=3, walks_per_node=4, subparts=1,
                     update_rule=1)
    V = orc.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    for ep in range(2):
        orc.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    assert orc.auc(orc.score_pairs(V, Cm, test), orc.score_pairs(V, Cm, neg)) > 0.9
