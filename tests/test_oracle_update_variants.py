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


# ---------------------------------------------------------------- NEXT-4 shared-negative mini-batch (D17)
def _grid_matrix(rng, n, d):
    # values on a 2^-12 grid, so x +- 2^-10 is exact in fp32 and the central
    # difference of the fp64 loss has no representation error
    return (rng.integers(-2048, 2048, (n, d)) / 4096.0).astype(np.float32)


def test_batch_gradient_matches_finite_differences(orc):
    """The batch loss gradient (or_batch_loss_grad) against central differences,
    on batches with repeated vertex rows, a context row that is both a positive
    and a shared negative, and a repeated negative (their gradients add)."""
    rng = np.random.default_rng(11)
    n, d = 12, 6
    for trial in range(6):
        V = _grid_matrix(rng, n, d)
        Cm = _grid_matrix(rng, n, d)
        B, Kp = int(rng.integers(1, 6)), int(rng.integers(0, 5))
        pairs = rng.integers(0, n, (B, 2)).astype(np.uint32)
        negs = rng.integers(0, n, Kp).astype(np.uint32)
        if trial % 2 and Kp:
            negs[0] = pairs[0, 1]            # positive context row reused as a negative
            pairs[-1, 0] = pairs[0, 0]       # repeated vertex row
        L, grads = orc.batch_loss_grad(V, Cm, pairs, negs)
        h = 2.0 ** -10
        for (kind, r), g in grads.items():
            M = V if kind == "v" else Cm
            for m in range(d):
                Mp, Mm = M.copy(), M.copy()
                Mp[r, m] += h
                Mm[r, m] -= h
                args_p = (Mp, Cm) if kind == "v" else (V, Mp)
                args_m = (Mm, Cm) if kind == "v" else (V, Mm)
                fd = (orc.batch_loss_grad(*args_p, pairs, negs)[0] - orc.batch_loss_grad(*args_m, pairs, negs)[0]) / (2 * h)
                assert abs(fd - g[m]) <= 1e-5 * max(1.0, abs(fd)), (kind, r, m, fd, g[m])
        # rows not in the batch have no gradient entry, and the keys are exactly the touched rows
        assert {k for k in grads if k[0] == "v"} == {("v", int(s)) for s in pairs[:, 0]}
        assert {k for k in grads if k[0] == "c"} == {("c", int(c)) for c in list(pairs[:, 1]) + list(negs)}


def test_batch_step_is_one_sgd_step(orc):
    rng = np.random.default_rng(12)
    n, d = 20, 8
    V = rng.normal(0, 0.3, (n, d)).astype(np.float32)
    Cm = rng.normal(0, 0.3, (n, d)).astype(np.float32)
    pairs = rng.integers(0, n, (5, 2)).astype(np.uint32)
    negs = rng.integers(0, n, 4).astype(np.uint32)
    L, grads = orc.batch_loss_grad(V, Cm, pairs, negs)
    V2, C2 = V.copy(), Cm.copy()
    L2 = orc.train_batch(V2, C2, pairs, negs, 0.05)
    assert L2 == L
    for (kind, r), g in grads.items():
        before, after = (V, V2) if kind == "v" else (Cm, C2)
        want = (before[r].astype(np.float64) - float(np.float32(0.05)) * g).astype(np.float32)  # eta = (double)lr
        assert np.array_equal(after[r], want)
    touched_v = {r for k, r in grads if k == "v"}
    for r in range(n):
        if r not in touched_v:
            assert np.array_equal(V2[r], V[r])


def test_batch_of_one_is_the_accumulated_rule(orc):
    """B = 1 with distinct rows: the mini-batch step is the accumulated-gradient
    update of that sample (same gradient; fp64 rounding order may differ)."""
    rng = np.random.default_rng(13)
    n, d = 30, 16
    for _ in range(20):
        V = rng.normal(0, 0.3, (n, d)).astype(np.float32)
        Cm = rng.normal(0, 0.3, (n, d)).astype(np.float32)
        ids = rng.permutation(n)[:6]
        s, dst, negs = int(ids[0]), int(ids[1]), ids[2:6].astype(np.uint32)
        V1, C1, V2, C2 = V.copy(), Cm.copy(), V.copy(), Cm.copy()
        l1 = orc.train_batch(V1, C1, np.array([[s, dst]], np.uint32), negs, 0.05)
        l2 = orc.train_sample_accumulated(V2, C2, s, dst, negs, 0.05)
        assert abs(l1 - l2) <= 1e-12 * abs(l2)
        assert np.abs(V1 - V2).max() <= 1e-7 and np.abs(C1 - C2).max() <= 1e-7


def test_batch_rule_epoch_equals_replay(orc):
    off, tgt = synth.rmat_graph(120, 700, 8)
    cfg = orc.Config(dim=16, negatives=7, walk_len=8, window=2, walks_per_node=1, episodes=1, subparts=2,
                     parts=2, seed=42, update_rule=2, batch=9)
    V = orc.init_vertex(120, 16, 42)
    Cm = np.zeros_like(V)
    V2, C2 = V.copy(), Cm.copy()
    ns, loss = orc.train_epoch(cfg, off, tgt, V, Cm, 2, 0.05)
    thr, al = orc.build_alias_tables(cfg, off)
    pb = orc.partition_bounds(0, 120, 2).astype(np.int64)
    pairs, boff = orc.build_episode(cfg, off, tgt, 2, 0)
    total, L = 0, 0.0
    for r in range(2):
        for t in range(2):
            for g in range(2):
                B = (((g - r) % 2) * 2 + t) * 2 + g
                blk = pairs[int(boff[B]):int(boff[B + 1])]
                for b0 in range(0, len(blk), 9):
                    negs = orc.batch_negatives(cfg, thr, al, int(pb[g]), int(pb[g + 1] - pb[g]), 2, 0, B, b0 // 9)
                    L += orc.train_batch(V2, C2, blk[b0:b0 + 9], negs, 0.05)
                    total += len(blk[b0:b0 + 9])
    assert ns == total and abs(loss - L) <= 1e-9 * abs(L)
    assert np.array_equal(V, V2) and np.array_equal(Cm, C2)


def test_batch_negatives_follow_the_alias_distribution(orc):
    # shared negatives come from the context part's deg^0.75 table (reading D9)
    off, tgt = synth.rmat_graph(50, 400, 9)
    cfg = orc.Config(dim=8, negatives=64, parts=1, update_rule=2, batch=128)
    thr, al = orc.build_alias_tables(cfg, off)
    deg = np.diff(off.astype(np.int64))
    w = deg.astype(np.float64) ** 0.75
    w /= w.sum()
    counts = np.zeros(50)
    for b in range(3000):
        for x in orc.batch_negatives(cfg, thr, al, 0, 50, 0, 0, 0, b):
            counts[int(x)] += 1
    tv = 0.5 * np.abs(counts / counts.sum() - w).sum()
    assert tv < 0.01, tv


def test_batch_rule_learns(orc):
    n = 600
    u, v = synth.planted_partition_edges(n, 6, 10.0, 0.5, 3)
    off, tgt, test = synth.split_edges(n, u, v, 0.1, 7)
    neg = synth.negative_pairs(n, u, v, len(test), 8)
    cfg = orc.Config(dim=32, negatives=16, walk_len=10, window=3, walks_per_node=2, episodes=1, subparts=2,
                     parts=1, seed=42, update_rule=2, batch=32)
    V = orc.init_vertex(n, 32, 42)
    Cm = np.zeros_like(V)
    for ep in range(4):
        orc.train_epoch(cfg, off, tgt, V, Cm, ep, 0.05)
    auc = orc.auc(orc.score_pairs(V, Cm, test), orc.score_pairs(V, Cm, neg))
    assert auc > 0.85, auc
